// nlfem_gpu2d.cu -- the reference's two-dimensional path (P1 triangles, disk
// kernel) on sm_100a: the n == 2 branches of nlfem::assemble
// (assembly.cpp:617-843 with et.n == 2; ball_approx.cpp:74-80, 104-108,
// 232-240, 273-281; geometry.cpp:59-71, 135-139; quadrature.cpp:17-21, 98-102).
//
// The 2D problems are small next to the 3D ones (C4 has 7e9 element pairs; a
// 2D mesh of 1e5 triangles has ~1e7), so this path is built for clarity and
// exact parity rather than for the last FLOP, and it carries the north star's
// reduction literally: every element pair emits its matrix and load-vector
// contributions as (key, value) entries with the reference's own keys
// (row << 32 | col for the upper triangle, row << 32 | 0xFFFFFFFF for the rhs,
// assembly.cpp:92-241), and one stable radix sort plus an in-order segmented
// sum -- a deterministic segmented reduction, no floating-point atomics --
// produces the upper-triangle stream that the CSR expansion mirrors, as the
// reference's merge tree does (assembly.cpp:767-833).
//
// Pipeline (one call of nlfem_gpu_assemble_2d):
//   k2_prep       quadrature points, spreads, grid keys per element
//   grid          elements sorted by cell (CUB radix sort) + cell starts
//   k2_pairs<0/1> CTA per interior (outer) element T: the candidates of the
//                 reach box, the reference's per-(T, q, T') decision for the
//                 three outer points (5-bit codes), BallExitsMesh probe; count
//                 pass, then fill in candidate order
//   k2_integrate  thread per element pair: the pieces (whole / Gauss sub-
//                 triangles / Monte Carlo caps), the per-point flush summed
//                 over the three points, 21 keyed entries
//   k2_fterm      thread per outer element: its load-vector f-term entries
//   sort + k2_segsum  CUB stable radix sort of the entries, in-order sums
//   k2_expand     upper triangle -> full symmetric CSR with sorted columns
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "geom.cuh"
#include "nlfem_gpu.h"
#include "nlfem_mc_stream.h"

namespace {

struct Fail2 {
  int code;
  std::string msg;
};

#define CK2(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw Fail2{NLFEM_GPU_ENODEVICE, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t m) {
    if (m <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    CK2(cudaMalloc(&p, std::max<size_t>(m, 1) * sizeof(T)));
    n = std::max<size_t>(m, 1);
  }
  void upload(const T* h, size_t m, cudaStream_t s) {
    ensure(m);
    if (m) CK2(cudaMemcpyAsync(p, h, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
};

constexpr int kMaxTerms2 = 32;
struct Poly2 {
  int n;
  double c[kMaxTerms2];
  int e[kMaxTerms2][3];
};

// Polynomial::eval (reference polynomial.cpp:28-37): per term c x^e0 y^e1 z^e2
// by repeated multiplication, terms summed in order
__device__ double poly2_eval(const Poly2& P, Vd p) {
  double acc = 0;
  for (int t = 0; t < P.n; ++t) {
    double v = P.c[t];
    for (int i = 0; i < P.e[t][0]; ++i) v *= p.x;
    for (int i = 0; i < P.e[t][1]; ++i) v *= p.y;
    for (int i = 0; i < P.e[t][2]; ++i) v *= p.z;
    acc += v;
  }
  return acc;
}

// the degree-2 triangle rule: edge midpoints, weights 1/3 (quadrature.cpp:17-21)
__device__ __forceinline__ double rb2(int k, int i) {
  // rows (0.5, 0.5, 0), (0, 0.5, 0.5), (0.5, 0, 0.5)
  return (k == 0) ? (i == 2 ? 0.0 : 0.5) : (k == 1 ? (i == 0 ? 0.0 : 0.5) : (i == 1 ? 0.0 : 0.5));
}
constexpr double kW2 = 1.0 / 3.0;

struct Dev2 {
  int K, J, KI, U;
  int strategy, mc;
  uint32_t k0, k1;
  double C, delta, slack, inside_cut, r2;
  const double* node;    // [3J]
  const int* verts;      // [3K]
  const int* nbr;        // [3K]
  const double* cen;     // [3K]
  const double* rad;     // [K]
  const double* vol;     // [K]
  const double* tau;     // [K] tau_vol(diam, 2), host std::pow
  const double* inv;     // [4K]
  const uint8_t* region;
  const int* interior;   // [KI]
  const int* dof;        // [J]
  const double* gnode;   // [J] g at constrained nodes
  double gox, goy, ginv, rmax;
  int gx, gy;
  int kshift;             // entry keys: row << kshift | col, col = U for the rhs
  const int* cell_start;  // [gx*gy + 1]
  const int* cell_elems;  // [K]
  Poly2 f, g;
};

__constant__ Dev2 c2;

__device__ __forceinline__ Vd node2(int v) {
  return {c2.node[3 * (long long)v], c2.node[3 * (long long)v + 1], c2.node[3 * (long long)v + 2]};
}
__device__ __forceinline__ void elem_verts2(int t, Vd v[3]) {
  for (int i = 0; i < 3; ++i) v[i] = node2(c2.verts[3 * (long long)t + i]);
}
// quadrature point k of the simplex v: p = b0 v0; p = p + b_i v_i
__device__ __forceinline__ Vd qpoint2(const Vd v[3], int k) {
  Vd p = vscale(rb2(k, 0), v[0]);
  for (int i = 1; i < 3; ++i) p = vadd(p, vscale(rb2(k, i), v[i]));
  return p;
}
// simplex_volume, n == 2 (geometry.cpp:60): 0.5 |cross(v1 - v0, v2 - v0)|
__device__ __forceinline__ double tri_area(Vd a, Vd b, Vd c) {
  return 0.5 * sqrt(vnorm2(vcross(vsub(b, a), vsub(c, a))));
}
// point_segment_distance (geometry.cpp:91-96)
__device__ __forceinline__ double seg_dist(Vd p, Vd a, Vd b) {
  const Vd d = vsub(b, a);
  const double len2 = vnorm2(d);
  double t = len2 > 0 ? vdot(vsub(p, a), d) / len2 : 0.0;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  return vdist(p, vadd(a, vscale(t, d)));
}
// distance_point_simplex, n == 2 (geometry.cpp:129-139 with barycentric 66-71)
__device__ double dist_point_tri(Vd p, const Vd v[3]) {
  const Vd e1 = vsub(v[1], v[0]), e2 = vsub(v[2], v[0]), b = vsub(p, v[0]);
  const double det = e1.x * e2.y - e1.y * e2.x;
  const double l1 = (b.x * e2.y - b.y * e2.x) / det;
  const double l2 = (e1.x * b.y - e1.y * b.x) / det;
  const double l0 = 1.0 - l1 - l2;
  if (!(l0 < 0) && !(l1 < 0) && !(l2 < 0)) return 0.0;
  double d = seg_dist(p, v[0], v[1]);
  d = fmin(d, seg_dist(p, v[1], v[2]));
  return fmin(d, seg_dist(p, v[2], v[0]));
}

enum : unsigned { k2None = 0, k2Whole = 1, k2OutCap = 2, k2Straddle = 16 };

__device__ __forceinline__ Vd pick3(const Vd v[3], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]);
}

// A straddling triangle in the reference's slot order (crossing_points,
// geometry.cpp:39-50: inside slots ascending, outside slots ascending,
// crossing k = i (3 - m) + o): m = 1 -> I0 | O0 O1, X0 = (I0,O0), X1 = (I0,O1);
// m = 2 -> I0 I1 | O0, X0 = (I0,O0), X1 = (I1,O0).  Vertices are picked by
// selects, so nothing is indexed at run time (all in registers).
struct Strad2 {
  int m;
  Vd I0, I1, O0, O1, X0, X1;
};
__device__ __forceinline__ Strad2 straddle2(const Vd v[3], unsigned mask, Vd xq) {
  Strad2 S;
  const unsigned om = ~mask & 7u;
  S.m = __popc(mask);
  const int i0 = __ffs(mask) - 1, o0 = __ffs(om) - 1, last = 3 - i0 - o0;
  S.I0 = pick3(v, i0);
  S.O0 = pick3(v, o0);
  if (S.m == 1) {
    S.O1 = pick3(v, last);
    S.I1 = S.I0;
  } else {
    S.I1 = pick3(v, last);
    S.O1 = S.O0;
  }
  const Vd a1 = S.m == 1 ? S.I0 : S.I1, b1 = S.m == 1 ? S.O1 : S.O0;
  const double t0 = edge_crossing(S.I0, S.O0, xq, c2.delta);
  S.X0 = vadd(S.I0, vscale(t0, vsub(S.O0, S.I0)));
  const double t1 = edge_crossing(a1, b1, xq, c2.delta);
  S.X1 = vadd(a1, vscale(t1, vsub(b1, a1)));
  return S;
}

// approxcaps, n == 2 (straddle_inner with sphere points, ball_approx.cpp:
// 210-229): the inside vertices, the two crossings and the sphere point of the
// crossing pair (it shares an inside or an outside vertex), then the
// reference's monotone-chain hull (hull2d, geometry.cpp:161-196: points sorted
// by (x, y), duplicates dropped, lower and upper chains with cross <= 0
// popped) and the fan from the centroid of the hull vertices summed in index
// order (triangulate_polytope, geometry.cpp:307-329).  Calls fn(a, b, c) for
// every fan piece above tau; returns the number of them (a degenerate hull
// has none: hull_pieces swallows DegenerateHull).
template <class Fn>
__device__ int approx_pieces2(const Strad2& S, Vd xq, double tau, Fn fn) {
  Vd P[5];
  int n = 0;
  P[n++] = S.I0;
  if (S.m == 2) P[n++] = S.I1;
  P[n++] = S.X0;
  P[n++] = S.X1;
  {
    const Vd mid = vsub(vscale(0.5, vadd(S.X0, S.X1)), xq);
    const double len = sqrt(vnorm2(mid));
    if (len > 0) P[n++] = vadd(xq, vscale(c2.delta / len, mid));
  }
  int idx[5];
  for (int i = 0; i < n; ++i) idx[i] = i;
  for (int i = 1; i < n; ++i) {  // insertion sort by (x, y), stable
    const int v = idx[i];
    int j = i - 1;
    while (j >= 0 && (P[idx[j]].x > P[v].x || (P[idx[j]].x == P[v].x && P[idx[j]].y > P[v].y))) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
  int u = 0;
  for (int i = 0; i < n; ++i)
    if (u == 0 || !(P[idx[u - 1]].x == P[idx[i]].x && P[idx[u - 1]].y == P[idx[i]].y))
      idx[u++] = idx[i];
  auto cr = [&](int o, int a, int b) {
    return (P[a].x - P[o].x) * (P[b].y - P[o].y) - (P[a].y - P[o].y) * (P[b].x - P[o].x);
  };
  int ring[10], k = 0;
  for (int i = 0; i < u; ++i) {
    while (k >= 2 && cr(ring[k - 2], ring[k - 1], idx[i]) <= 0) --k;
    ring[k++] = idx[i];
  }
  for (int i = u - 1, t = k + 1; i-- > 0;) {
    while (k >= t && cr(ring[k - 2], ring[k - 1], idx[i]) <= 0) --k;
    ring[k++] = idx[i];
  }
  if (k < 4) return 0;
  const int nr = k - 1;
  // centroid of the hull vertices, summed in ascending point index
  unsigned used = 0;
  for (int i = 0; i < nr; ++i) used |= 1u << ring[i];
  Vd c = {0, 0, 0};
  int nv = 0;
  for (int i = 0; i < n; ++i)
    if (used >> i & 1u) {
      c = vadd(c, P[i]);
      ++nv;
    }
  c = vscale(1.0 / double(nv), c);
  int kept = 0;
  for (int i = 0; i < nr; ++i) {
    const Vd a = P[ring[i]], b = P[ring[(i + 1) % nr]];
    if (tri_area(c, a, b) > tau) {
      fn(c, a, b);
      ++kept;
    }
  }
  return kept;
}

// does the straddler emit a piece (push_piece's volume floor, ball_approx.cpp:
// 141; straddle_inner / straddle_outer n == 2, 232-240 / 273-281)?  An item
// without pieces never reaches the sink: no flush, no pattern keys.
__device__ bool straddle_kept2(const Vd v[3], unsigned mask, Vd xq, double tau, bool outer) {
  const Strad2 S = straddle2(v, mask, xq);
  if (S.m == 1) {
    if (tri_area(S.I0, S.X0, S.X1) > tau) return true;
  } else {
    if (tri_area(S.I0, S.I1, S.X1) > tau) return true;
    if (tri_area(S.I0, S.X1, S.X0) > tau) return true;
  }
  if (!outer) return false;
  if (S.m == 1) return tri_area(S.O0, S.O1, S.X1) > tau || tri_area(S.O0, S.X1, S.X0) > tau;
  return tri_area(S.O0, S.X0, S.X1) > tau;
}

// The reference's per-(T, q, T') decision (assembly.cpp:722-760), n == 2.
__device__ unsigned decide2(Vd xq, int t) {
  const double delta = c2.delta;
  const Vd ct = {c2.cen[3 * (long long)t], c2.cen[3 * (long long)t + 1], c2.cen[3 * (long long)t + 2]};
  const double gap = vdist(ct, xq);
  const double r = c2.rad[t];
  if (gap >= r + delta) return k2None;
  const int S = c2.strategy;
  if (S == NLFEM_STRATEGY_BARYCENTER) return gap < delta ? k2Whole : k2None;
  Vd v[3];
  elem_verts2(t, v);
  if (S == NLFEM_STRATEGY_OVERLAP)
    return (gap + r < delta || dist_point_tri(xq, v) < delta) ? k2Whole : k2None;
  if (gap + r < c2.inside_cut) return k2Whole;
  // classify_simplex (geometry.cpp:8-24)
  const double r_in = delta - 1e-10 * delta;
  const double rr = r_in * r_in;
  unsigned mask = 0;
  for (int i = 0; i < 3; ++i)
    if (vnorm2(vsub(v[i], xq)) < rr) mask |= 1u << i;
  if (mask == 7u) return k2Whole;
  if (mask != 0) {
    if (S == NLFEM_STRATEGY_INSIDE) return k2None;
    if (S == NLFEM_STRATEGY_APPROXCAPS) {
      const Strad2 Sd = straddle2(v, mask, xq);
      return approx_pieces2(Sd, xq, c2.tau[t], [](Vd, Vd, Vd) {}) > 0 ? (k2Straddle | mask)
                                                                       : k2None;
    }
    return straddle_kept2(v, mask, xq, c2.tau[t], S == NLFEM_STRATEGY_FULLCAPS)
               ? (k2Straddle | mask)
               : k2None;
  }
  if (S == NLFEM_STRATEGY_FULLCAPS && dist_point_tri(xq, v) < delta) return k2OutCap;
  return k2None;
}

// ---- grid -------------------------------------------------------------------

__global__ void k2_cellkey(int K, unsigned* key, int* idx) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const double x = c2.cen[3 * (long long)t], y = c2.cen[3 * (long long)t + 1];
  int cx = (int)floor((x - c2.gox) * c2.ginv), cy = (int)floor((y - c2.goy) * c2.ginv);
  cx = cx < 0 ? 0 : (cx >= c2.gx ? c2.gx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= c2.gy ? c2.gy - 1 : cy);
  key[t] = (unsigned)(cy * c2.gx + cx);
  idx[t] = t;
}

// start[c] = first sorted position with key >= c, for c = 0 .. ncell
__global__ void k2_cellstart(int K, int ncell, const unsigned* skey, int* start) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > K) return;
  const long long from = i == 0 ? 0 : (long long)skey[i - 1] + 1;
  const long long to = i == K ? ncell : (long long)skey[i];
  for (long long c = from; c <= to; ++c) start[c] = i;
}

// ---- element pairs ----------------------------------------------------------

constexpr int kP2Threads = 128;

// CTA per outer element.  MODE 0 counts its pairs, MODE 1 writes them (partner,
// 15-bit code: 5 bits per outer point) in candidate order: grid rows of the
// reach box, cells along x, element ids ascending within a cell.
template <int MODE>
__global__ void __launch_bounds__(kP2Threads) k2_pairs(const long long* off, int* cnt,
                                                       int* partner, unsigned* code,
                                                       int* err_elem) {
  const int ii = blockIdx.x;
  if (ii >= c2.KI) return;
  const int T = c2.interior[ii];
  Vd v[3];
  elem_verts2(T, v);
  Vd xq[3];
  for (int k = 0; k < 3; ++k) xq[k] = qpoint2(v, k);
  const Vd cT = {c2.cen[3 * (long long)T], c2.cen[3 * (long long)T + 1], c2.cen[3 * (long long)T + 2]};
  double spread = 0;
  for (int k = 0; k < 3; ++k) spread = fmax(spread, vdist(xq[k], cT));
  const double reach = c2.delta + spread + c2.rmax;
  auto cell = [](double x, double o, int n) {
    int c = (int)floor((x - o) * c2.ginv);
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
  };
  const int x0 = cell(cT.x - reach, c2.gox, c2.gx), x1 = cell(cT.x + reach, c2.gox, c2.gx);
  const int y0 = cell(cT.y - reach, c2.goy, c2.gy), y1 = cell(cT.y + reach, c2.goy, c2.gy);
  __shared__ int wbase[kP2Threads / 32 + 1];
  int total = 0;  // pairs written so far (same in every thread)
  const long long o = MODE ? off[ii] : 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int y = y0; y <= y1; ++y) {
    const int a = c2.cell_start[y * c2.gx + x0], b = c2.cell_start[y * c2.gx + x1 + 1];
    for (int base = a; base < b; base += kP2Threads) {
      const int k = base + threadIdx.x;
      unsigned cd = 0;
      int Tp = -1;
      if (k < b) {
        Tp = c2.cell_elems[k];
        for (int q = 0; q < 3; ++q) {
          unsigned c = decide2(xq[q], Tp);
          cd |= c << (5 * q);
        }
        // BallExitsMesh (assembly.cpp:710-719): an unglued facet of a reached
        // element closer than delta - slack to an outer point
        for (int f = 0; f < 3; ++f) {
          if (c2.nbr[3 * (long long)Tp + f] >= 0) continue;
          Vd w[3];
          elem_verts2(Tp, w);
          // facet opposite slot f: the other two vertices in slot order
          const Vd fa = w[f == 0 ? 1 : 0], fb = w[f == 2 ? 1 : 2];
          for (int q = 0; q < 3; ++q)
            if (seg_dist(xq[q], fa, fb) < c2.delta - c2.slack) atomicMin(err_elem, Tp);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, cd != 0);
      if (lane == 0) wbase[wid] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < kP2Threads / 32; ++w) {
        before += w < wid ? wbase[w] : 0;
        tot += wbase[w];
      }
      if (MODE && cd) {
        const long long pos = o + total + before + __popc(bal & ((1u << lane) - 1));
        partner[pos] = Tp;
        code[pos] = cd;
      }
      total += tot;
      __syncthreads();
    }
  }
  if (!MODE && threadIdx.x == 0) cnt[ii] = total;
}

// ---- integration --------------------------------------------------------------

// per-parent moment sums (AsmSink, assembly.cpp:257-370)
struct Acc2 {
  double S0, Sg, S1[3], S2[3][3];
  __device__ void zero() {
    S0 = Sg = 0;
    for (int i = 0; i < 3; ++i) {
      S1[i] = 0;
      for (int j = 0; j < 3; ++j) S2[i][j] = 0;
    }
  }
};

// accumulate_point (assembly.cpp:332-344): bary via inv_edges (ball_approx.cpp:104-108)
__device__ __forceinline__ void acc_point2(Acc2& A, int t, bool cons, Vd y, double w,
                                           Vd v0) {
  A.S0 += w;
  if (cons) {
    A.Sg += w * poly2_eval(c2.g, y);
    return;
  }
  const double* inv = c2.inv + 4 * (long long)t;
  const Vd d = vsub(y, v0);
  double b[3];
  b[1] = inv[0] * d.x + inv[1] * d.y;
  b[2] = inv[2] * d.x + inv[3] * d.y;
  b[0] = 1.0 - b[1] - b[2];
  for (int i = 0; i < 3; ++i) {
    const double wb = w * b[i];
    A.S1[i] += wb;
    for (int j = 0; j < 3; ++j) A.S2[i][j] += wb * b[j];
  }
}

// sub (assembly.cpp:372-381): the degree-2 rule on a sub-triangle
__device__ __forceinline__ void sub2(Acc2& A, int t, bool cons, const Vd s[3], Vd v0) {
  const double vol = tri_area(s[0], s[1], s[2]);
  for (int k = 0; k < 3; ++k) acc_point2(A, t, cons, qpoint2(s, k), vol * kW2, v0);
}

// cap (assembly.cpp:383-399) with the 2D Philox stream (include/nlfem_mc_stream.h)
__device__ __forceinline__ void cap2(Acc2& A, int t, bool cons, const Vd s[3], Vd v0, Vd xq, uint32_t T,
                     uint32_t q, uint32_t sub, unsigned long long& draws,
                     unsigned long long& hits) {
  const int M = c2.mc;
  const double w = tri_area(s[0], s[1], s[2]) / M;
  const double sv[3][3] = {{s[0].x, s[0].y, s[0].z}, {s[1].x, s[1].y, s[1].z},
                           {s[2].x, s[2].y, s[2].z}};
  uint32_t W[4];
  for (int k = 0; k < M; ++k) {
    if ((k & 1) == 0) nlfem_mc2_block(c2.k0, c2.k1, T, (uint32_t)t, q, sub, (uint32_t)(k >> 1), W);
    double y3[3];
    nlfem_mc2_sample(W, k & 1, sv[0], sv[1], sv[2], y3);
    const Vd y = {y3[0], y3[1], y3[2]};
    ++draws;
    if (vnorm2(vsub(y, xq)) >= c2.r2) continue;
    ++hits;
    acc_point2(A, t, cons, y, w, v0);
  }
}

constexpr int kEnt = 21;  // entries per pair: the upper triangle of <= 6 union nodes

// Entry keys, the reference's (row, col) order in as few bits as the system
// needs (the radix sort only sorts those): row << kshift | col with col = U
// standing for the reference's rhs column 0xFFFFFFFF; the sentinel of an
// unused slot, row = U, sorts after every real key.
__device__ __forceinline__ unsigned long long kmat(unsigned r, unsigned c) {
  return ((unsigned long long)r << c2.kshift) | c;
}
__device__ __forceinline__ unsigned long long krhs(unsigned r) { return kmat(r, (unsigned)c2.U); }
__device__ __forceinline__ unsigned long long ksent() { return kmat((unsigned)c2.U, (unsigned)c2.U); }

__device__ __forceinline__ void put2(unsigned long long* keys, double* vals, long long base,
                                     int& ne, unsigned long long key, double v) {
  keys[base + ne] = key;
  vals[base + ne] = v;
  ++ne;
}

// add_pair (assembly.cpp:401-411) as keyed entries
__device__ __forceinline__ void add_pair2(unsigned long long* keys, double* vals, long long base,
                                          int& ne, int dof_a, int node_a, int dof_b, int node_b,
                                          double v) {
  if (dof_a >= 0 && dof_b >= 0) {
    const unsigned long long lo = (unsigned)min(dof_a, dof_b), hi = (unsigned)max(dof_a, dof_b);
    put2(keys, vals, base, ne, kmat((unsigned)lo, (unsigned)hi), v);
  } else if (dof_a >= 0) {
    put2(keys, vals, base, ne, krhs((unsigned)dof_a),
         -v * c2.gnode[node_b]);
  } else if (dof_b >= 0) {
    put2(keys, vals, base, ne, krhs((unsigned)dof_b),
         -v * c2.gnode[node_a]);
  }
}

// thread per element pair (T, T'): the three points' pieces and flushes
// (whole / straddle_inner / straddle_outer / cap, flush: assembly.cpp:413-473),
// the per-point flush values summed over the points into one entry per node pair
__global__ void k2_integrate(long long npairs, const long long* off, const int* partner,
                             const unsigned* code, unsigned long long* keys, double* vals,
                             unsigned long long* stats) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long draws = 0, hits = 0, items = 0;
  if (p < npairs) {
    // outer element of the pair: binary search in the pair offsets
    int lo = 0, hi = c2.KI - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int T = c2.interior[lo];
    const int Tp = partner[p];
    const unsigned cd = code[p];
    Vd vT[3], vP[3];
    elem_verts2(T, vT);
    elem_verts2(Tp, vP);
    const double volT = c2.vol[T];
    const bool cons = c2.region[Tp] != 0;
    int nT[3], dT[3], nP[3];
    for (int a = 0; a < 3; ++a) {
      nT[a] = c2.verts[3 * (long long)T + a];
      dT[a] = c2.dof[nT[a]];
      nP[a] = c2.verts[3 * (long long)Tp + a];
    }
    // union U (flush, assembly.cpp:430-450) in fixed slots: 0-2 the outer
    // element's nodes, 3-5 the partner's nodes, active when not shared (the
    // order of a pair's entries does not matter: each key occurs once per pair)
    int un[6], ud[6], ms[6];
    bool act[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int m = -1;
#pragma unroll
      for (int j = 2; j >= 0; --j) m = nP[j] == nT[a] ? j : m;
      un[a] = nT[a];
      ud[a] = dT[a];
      ms[a] = m;
      act[a] = true;
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      bool shared = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) shared |= nT[a] == nP[j];
      un[3 + j] = nP[j];
      ud[3 + j] = c2.dof[nP[j]];
      ms[3 + j] = j;
      act[3 + j] = !shared;
    }
    double V[6][6];
#pragma unroll
    for (int x = 0; x < 6; ++x)
#pragma unroll
      for (int y = 0; y < 6; ++y) V[x][y] = 0;
    double rhsT[3] = {0, 0, 0};
    const double tauP = c2.tau[Tp];
    for (int q = 0; q < 3; ++q) {
      const unsigned c = (cd >> (5 * q)) & 31u;
      if (!c) continue;
      ++items;
      const Vd xq = qpoint2(vT, q);
      const double wN = kW2 * volT;  // rule.w[k] * vol (assembly.cpp:702)
      Acc2 A;
      A.zero();
      if (c == k2Whole) {
        const double vol = c2.vol[Tp];
        if (cons) {
          A.S0 += vol;
          for (int k = 0; k < 3; ++k) A.Sg += vol * kW2 * poly2_eval(c2.g, qpoint2(vP, k));
        } else {
          // whole (assembly.cpp:361-369), n == 2
          A.S0 += vol;
          const double s1 = vol / 3.0;
          const double offd = vol / double(3 * 4);
          for (int i = 0; i < 3; ++i) {
            A.S1[i] += s1;
            for (int j = 0; j < 3; ++j) A.S2[i][j] += offd * (i == j ? 2.0 : 1.0);
          }
        }
      } else if (c == k2OutCap) {
        // the whole element as one Monte Carlo region (assembly.cpp:754-759)
        cap2(A, Tp, cons, vP, vP[0], xq, (uint32_t)T, (uint32_t)q, 0u, draws, hits);
      } else {
        const Strad2 Sd = straddle2(vP, c & 7u, xq);
        if (c2.strategy == NLFEM_STRATEGY_APPROXCAPS) {
          approx_pieces2(Sd, xq, tauP, [&](Vd a, Vd b, Vd cc) {
            const Vd s[3] = {a, b, cc};
            sub2(A, Tp, cons, s, vP[0]);
          });
        } else if (Sd.m == 1) {  // straddle_inner, n == 2 (ball_approx.cpp:232-240)
          const Vd s[3] = {Sd.I0, Sd.X0, Sd.X1};
          if (tri_area(s[0], s[1], s[2]) > tauP) sub2(A, Tp, cons, s, vP[0]);
        } else {
          const Vd s1[3] = {Sd.I0, Sd.I1, Sd.X1};
          if (tri_area(s1[0], s1[1], s1[2]) > tauP) sub2(A, Tp, cons, s1, vP[0]);
          const Vd s2[3] = {Sd.I0, Sd.X1, Sd.X0};
          if (tri_area(s2[0], s2[1], s2[2]) > tauP) sub2(A, Tp, cons, s2, vP[0]);
        }
        if (c2.strategy == NLFEM_STRATEGY_FULLCAPS) {
          // straddle_outer, n == 2 (ball_approx.cpp:273-281): the kept pieces
          // in order, each a Monte Carlo region (sub index = kept order)
          uint32_t kept = 0;
          const Vd s1[3] = {Sd.O0, Sd.m == 1 ? Sd.O1 : Sd.X0, Sd.X1};
          if (tri_area(s1[0], s1[1], s1[2]) > tauP)
            cap2(A, Tp, cons, s1, vP[0], xq, (uint32_t)T, (uint32_t)q, kept++, draws, hits);
          if (Sd.m == 1) {
            const Vd s2[3] = {Sd.O0, Sd.X1, Sd.X0};
            if (tri_area(s2[0], s2[1], s2[2]) > tauP)
              cap2(A, Tp, cons, s2, vP[0], xq, (uint32_t)T, (uint32_t)q, kept++, draws, hits);
          }
        }
      }
      // flush (assembly.cpp:413-473) into the per-pair sums
      const double C = c2.C;
      if (cons) {
        const double base = wN * 2.0 * C;
        for (int a = 0; a < 3; ++a) {
          rhsT[a] += base * A.Sg * rb2(q, a);
          for (int b = a; b < 3; ++b) V[a][b] += base * A.S0 * rb2(q, a) * rb2(q, b);
        }
      } else {
        // the moments by union slot through selects (static indices: the
        // accumulators stay in registers)
        double s1u[6];
#pragma unroll
        for (int x = 0; x < 6; ++x) {
          s1u[x] = 0;
#pragma unroll
          for (int i = 0; i < 3; ++i) s1u[x] = ms[x] == i ? A.S1[i] : s1u[x];
        }
        const double scale = C * wN;
#pragma unroll
        for (int x = 0; x < 6; ++x) {
          const double cx = x < 3 ? rb2(q, x) : 0.0;
#pragma unroll
          for (int y = x; y < 6; ++y) {
            const double cy = y < 3 ? rb2(q, y) : 0.0;
            double s2 = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int j = 0; j < 3; ++j) s2 = (ms[x] == i && ms[y] == j) ? A.S2[i][j] : s2;
            V[x][y] += scale * (s2 - cx * s1u[y] - cy * s1u[x] + cx * cy * A.S0);
          }
        }
      }
    }
    // the pair's entries (a fixed slot range; unused slots carry the sentinel key)
    const long long base = p * kEnt;
    int ne = 0;
    if (cons) {
      for (int a = 0; a < 3; ++a) {
        if (dT[a] >= 0)
          put2(keys, vals, base, ne, krhs((unsigned)dT[a]),
               rhsT[a]);
        for (int b = a; b < 3; ++b) add_pair2(keys, vals, base, ne, dT[a], nT[a], dT[b], nT[b], V[a][b]);
      }
    } else {
#pragma unroll
      for (int x = 0; x < 6; ++x)
#pragma unroll
        for (int y = x; y < 6; ++y)
          if (act[x] && act[y]) add_pair2(keys, vals, base, ne, ud[x], un[x], ud[y], un[y], V[x][y]);
    }
    for (; ne < kEnt; ++ne) {
      keys[base + ne] = ksent();
      vals[base + ne] = 0;
    }
  }
  for (int s = 16; s > 0; s >>= 1) {
    draws += __shfl_xor_sync(0xffffffffu, draws, s);
    hits += __shfl_xor_sync(0xffffffffu, hits, s);
    items += __shfl_xor_sync(0xffffffffu, items, s);
  }
  if ((threadIdx.x & 31) == 0) {
    if (draws) atomicAdd(stats, draws);
    if (hits) atomicAdd(stats + 1, hits);
    if (items) atomicAdd(stats + 2, items);
  }
}

// load-vector f-term (assembly.cpp:703-709): rhs[dof_a] += w c_a f(x_q), summed
// over the three points, one entry per node of the outer element
__global__ void k2_fterm(long long base0, unsigned long long* keys, double* vals) {
  const int ii = blockIdx.x * blockDim.x + threadIdx.x;
  if (ii >= c2.KI) return;
  const int T = c2.interior[ii];
  Vd v[3];
  elem_verts2(T, v);
  const double vol = c2.vol[T];
  double r[3] = {0, 0, 0};
  for (int q = 0; q < 3; ++q) {
    const Vd xq = qpoint2(v, q);
    const double w = kW2 * vol;
    const double fv = poly2_eval(c2.f, xq);
    for (int a = 0; a < 3; ++a) r[a] += w * rb2(q, a) * fv;
  }
  for (int a = 0; a < 3; ++a) {
    const int d = c2.dof[c2.verts[3 * (long long)T + a]];
    const long long o = base0 + 3LL * ii + a;
    keys[o] = d >= 0 ? krhs((unsigned)d) : ksent();
    vals[o] = r[a];
  }
}

// ---- segmented reduction and CSR expansion --------------------------------------

__global__ void k2_flag(long long n, const unsigned long long* k, int* flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (k[i] != ksent() && (i == 0 || k[i] != k[i - 1])) ? 1 : 0;
}

// thread per distinct key: its entries summed in sorted (stable) order
__global__ void k2_segsum(long long n, const unsigned long long* k, const double* v,
                          const int* flag, const long long* uid, unsigned long long* uk,
                          double* uv) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  double s = v[i];
  for (long long j = i + 1; j < n && k[j] == k[i]; ++j) s += v[j];
  uk[uid[i]] = k[i];
  uv[uid[i]] = s;
}

// upper-triangle stream -> full CSR entries (row << 32 | col) incl. mirrors;
// rhs entries go to rhs[row]
__global__ void k2_mirror(long long nu, const unsigned long long* uk, const double* uv,
                          unsigned long long* fk, double* fv, int* fflag, double* rhs) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  const unsigned long long key = uk[i];
  const unsigned r = (unsigned)(key >> c2.kshift),
                 c = (unsigned)(key & ((1ull << c2.kshift) - 1));
  if (c == (unsigned)c2.U) {
    rhs[r] = uv[i];
    fflag[2 * i] = fflag[2 * i + 1] = 0;
    fk[2 * i] = fk[2 * i + 1] = ksent();
    return;
  }
  fk[2 * i] = key;
  fv[2 * i] = uv[i];
  fflag[2 * i] = 1;
  if (r != c) {
    fk[2 * i + 1] = kmat(c, r);
    fv[2 * i + 1] = uv[i];
    fflag[2 * i + 1] = 1;
  } else {
    fk[2 * i + 1] = ksent();
    fflag[2 * i + 1] = 0;
  }
}

__global__ void k2_csr(long long n, const unsigned long long* fk, const double* fv,
                       int* rowcnt, int* col, double* val) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long key = fk[i];
  col[i] = (int)(key & ((1ull << c2.kshift) - 1));
  val[i] = fv[i];
  atomicAdd(rowcnt + (int)(key >> c2.kshift), 1);
}

unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }

__global__ void k2_widen(long long n, const int* in, long long* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i + 1] = in[i];
}

// exclusive scan of n ints into out[0..n] (out[n] = total)
void xscan(const int* in, long long* out, long long n, cudaStream_t st, Buf<unsigned char>& tmp) {
  CK2(cudaMemsetAsync(out, 0, sizeof(long long), st));
  if (n <= 0) return;
  k2_widen<<<nb(n, 256), 256, 0, st>>>(n, in, out);
  size_t bytes = 0;
  CK2(cub::DeviceScan::InclusiveSum(nullptr, bytes, out + 1, out + 1, n, st));
  tmp.ensure(bytes);
  CK2(cub::DeviceScan::InclusiveSum(tmp.p, bytes, out + 1, out + 1, n, st));
}

template <class T>
T read1(const T* d, cudaStream_t st) {
  T h{};
  CK2(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  CK2(cudaStreamSynchronize(st));
  return h;
}

void poly2_from(const nlfem_gpu_poly* p, Poly2& d) {
  if (!p || p->nterms < 0 || p->nterms > kMaxTerms2)
    throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: polynomial with too many terms"};
  d.n = p->nterms;
  for (int t = 0; t < d.n; ++t) {
    d.c[t] = p->coef[t];
    for (int a = 0; a < 3; ++a) d.e[t][a] = p->exps[3 * t + a];
  }
}

double poly2_host(const Poly2& P, const double* x) {
  double acc = 0;
  for (int t = 0; t < P.n; ++t) {
    double v = P.c[t];
    for (int i = 0; i < P.e[t][0]; ++i) v *= x[0];
    for (int i = 0; i < P.e[t][1]; ++i) v *= x[1];
    for (int i = 0; i < P.e[t][2]; ++i) v *= x[2];
    acc += v;
  }
  return acc;
}

void assemble2d(const nlfem_gpu_mesh2d* m, const nlfem_gpu_dofs* dofs,
                const nlfem_gpu_kernel* k, const nlfem_gpu_poly* f, const nlfem_gpu_poly* g,
                const nlfem_gpu_config* cfg, nlfem_gpu_csr* out, nlfem_gpu_stats* stats) {
  const auto wall0 = std::chrono::steady_clock::now();
  if (!(k->delta > 0)) throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: delta must be positive"};
  if (cfg->mc_samples <= 0) throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: mc_samples must be positive"};
  if (cfg->strategy < 0 || cfg->strategy > NLFEM_STRATEGY_FULLCAPS)
    throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: unknown strategy"};
  int dev = cfg->device;
  if (dev < 0) CK2(cudaGetDevice(&dev));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Fail2{NLFEM_GPU_ENODEVICE, "no CUDA device"};
  // one 2D call per device at a time: the parameter block c2 is per device
  static std::mutex locks_mu;
  static std::map<int, std::mutex> locks;
  std::mutex* dmu;
  {
    std::lock_guard<std::mutex> g(locks_mu);
    dmu = &locks[dev];
  }
  std::lock_guard<std::mutex> dev_lock(*dmu);
  int prev = 0;
  CK2(cudaGetDevice(&prev));
  CK2(cudaSetDevice(dev));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev};
  int major = 0;
  CK2(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) throw Fail2{NLFEM_GPU_ENODEVICE, "device is not sm_100 class (built for sm_100a only)"};
  cudaStream_t st;
  CK2(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  cudaEvent_t e0, e1, ep[3];
  CK2(cudaEventCreate(&e0));
  CK2(cudaEventCreate(&e1));
  for (auto& e : ep) CK2(cudaEventCreate(&e));
  struct EventGuard {  // released on every exit path (exceptions included)
    cudaEvent_t* e;
    ~EventGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t evs[5] = {e0, e1, ep[0], ep[1], ep[2]};
  EventGuard eguard{evs};

  const int K = m->elem_count, J = m->node_count;
  Dev2 D{};
  D.K = K;
  D.J = J;
  D.strategy = cfg->strategy;
  D.mc = cfg->mc_samples;
  D.k0 = (uint32_t)(cfg->seed & 0xffffffffu);
  D.k1 = (uint32_t)(cfg->seed >> 32);
  D.C = k->C;
  D.delta = k->delta;
  D.slack = 1e-10 * k->delta;                            // eps_geo (core.hpp:83)
  D.inside_cut = k->delta - D.slack - 1e-12 * k->delta;  // assembly.cpp:659
  D.r2 = k->delta * k->delta;
  poly2_from(f, D.f);
  poly2_from(g, D.g);
  // host-side setup of the call (the reference's assemble() does the same
  // before its workers start): interior list, g at the constrained nodes,
  // tau_vol with std::pow, grid geometry
  std::vector<int> interior;
  for (int t = 0; t < K; ++t)
    if (!m->region[t]) interior.push_back(t);
  D.KI = (int)interior.size();
  D.U = dofs->unknowns;
  int kbits = 1;
  while ((1LL << kbits) <= (long long)D.U) ++kbits;  // col in [0, U]
  D.kshift = kbits;
  const int key_bits = 2 * kbits;                      // row in [0, U] too
  std::vector<double> gnode(J, 0.0), tau(K);
  for (int v = 0; v < J; ++v)
    if (dofs->dof_of_node[v] < 0) gnode[v] = poly2_host(D.g, m->node_xyz + 3 * (size_t)v);
  double rmax = 0, xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300, asum = 0;
  for (int t = 0; t < K; ++t) {
    tau[t] = 1e-14 * std::pow(m->diam[t], 2);  // tau_vol(diam, 2) (core.hpp:85)
    rmax = std::max(rmax, m->radius[t]);
    xmin = std::min(xmin, m->center[3 * (size_t)t]);
    xmax = std::max(xmax, m->center[3 * (size_t)t]);
    ymin = std::min(ymin, m->center[3 * (size_t)t + 1]);
    ymax = std::max(ymax, m->center[3 * (size_t)t + 1]);
    asum += m->volume[t];
  }
  const double cellw = K ? std::max(std::sqrt(2.0 * asum / K), 1e-300) : 1.0;
  D.rmax = rmax;
  D.gox = xmin - 0.5 * cellw;
  D.goy = ymin - 0.5 * cellw;
  D.ginv = 1.0 / cellw;
  D.gx = std::max(1, (int)((xmax - D.gox) / cellw) + 2);
  D.gy = std::max(1, (int)((ymax - D.goy) / cellw) + 2);
  const long long ncell = (long long)D.gx * D.gy;

  Buf<double> node, cen, rad, vol, tau_d, inv, gn;
  Buf<int> verts, nbr, inter, dof;
  Buf<uint8_t> region;
  node.upload(m->node_xyz, 3 * (size_t)J, st);
  verts.upload(m->verts, 3 * (size_t)K, st);
  nbr.upload(m->neighbor, 3 * (size_t)K, st);
  cen.upload(m->center, 3 * (size_t)K, st);
  rad.upload(m->radius, K, st);
  vol.upload(m->volume, K, st);
  tau_d.upload(tau.data(), K, st);
  inv.upload(m->inv_edges, 4 * (size_t)K, st);
  region.upload(m->region, K, st);
  inter.upload(interior.data(), interior.size(), st);
  dof.upload(dofs->dof_of_node, J, st);
  gn.upload(gnode.data(), J, st);
  D.node = node.p;
  D.verts = verts.p;
  D.nbr = nbr.p;
  D.cen = cen.p;
  D.rad = rad.p;
  D.vol = vol.p;
  D.tau = tau_d.p;
  D.inv = inv.p;
  D.region = region.p;
  D.interior = inter.p;
  D.dof = dof.p;
  D.gnode = gn.p;
  Buf<int> cstart, celems, cidx;
  Buf<unsigned> ckey, ckey2;
  cstart.ensure(ncell + 1);
  celems.ensure(K);
  D.cell_start = cstart.p;
  D.cell_elems = celems.p;
  CK2(cudaMemcpyToSymbolAsync(c2, &D, sizeof(Dev2), 0, cudaMemcpyHostToDevice, st));
  CK2(cudaEventRecord(e0, st));
  Buf<unsigned char> tmp;
  // grid: elements sorted by cell (stable: ids ascending within a cell)
  ckey.ensure(K);
  ckey2.ensure(K);
  cidx.ensure(K);
  if (K > 0) {
    k2_cellkey<<<nb(K, 256), 256, 0, st>>>(K, ckey.p, cidx.p);
    size_t bytes = 0;
    CK2(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ckey.p, ckey2.p, cidx.p, celems.p, K, 0,
                                        32, st));
    tmp.ensure(bytes);
    CK2(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, ckey.p, ckey2.p, cidx.p, celems.p, K, 0,
                                        32, st));
  }
  k2_cellstart<<<nb(K + 1, 256), 256, 0, st>>>(K, (int)ncell, ckey2.p, cstart.p);
  // element pairs: count, scan, fill
  const int KI = D.KI;
  Buf<int> pcnt, err;
  Buf<long long> poff;
  pcnt.ensure(KI + 1);
  poff.ensure(KI + 1);
  err.ensure(1);
  const int big = 0x7fffffff;
  CK2(cudaMemcpyAsync(err.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  if (KI > 0) k2_pairs<0><<<KI, kP2Threads, 0, st>>>(nullptr, pcnt.p, nullptr, nullptr, err.p);
  xscan(pcnt.p, poff.p, KI, st, tmp);
  const long long npairs = read1(poff.p + KI, st);
  const int err_h = read1(err.p, st);
  if (err_h != big)
    throw Fail2{NLFEM_GPU_BALL_EXITS_MESH,
                "BallExitsMesh: ball reaches past an unglued facet of element " +
                    std::to_string(err_h)};
  Buf<int> partner;
  Buf<unsigned> code;
  partner.ensure(npairs + 1);
  code.ensure(npairs + 1);
  if (KI > 0) k2_pairs<1><<<KI, kP2Threads, 0, st>>>(poff.p, nullptr, partner.p, code.p, err.p);
  CK2(cudaEventRecord(ep[0], st));
  // integration: keyed entries
  const long long nent = npairs * kEnt + 3LL * KI;
  Buf<unsigned long long> keys, skeys, ukeys;
  Buf<double> vals, svals, uvals;
  Buf<unsigned long long> cnt;
  keys.ensure(nent + 1);
  vals.ensure(nent + 1);
  cnt.ensure(4);
  CK2(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), st));
  if (npairs > 0)
    k2_integrate<<<nb(npairs, 128), 128, 0, st>>>(npairs, poff.p, partner.p, code.p, keys.p,
                                                   vals.p, cnt.p);
  if (KI > 0) k2_fterm<<<nb(KI, 128), 128, 0, st>>>(npairs * kEnt, keys.p, vals.p);
  CK2(cudaEventRecord(ep[1], st));
  // deterministic segmented reduction: stable radix sort, in-order sums
  skeys.ensure(nent + 1);
  svals.ensure(nent + 1);
  if (nent > 0) {
    size_t bytes = 0;
    CK2(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, skeys.p, vals.p, svals.p, nent, 0,
                                        key_bits, st));
    tmp.ensure(bytes);
    CK2(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, skeys.p, vals.p, svals.p, nent, 0,
                                        key_bits, st));
  }
  Buf<int> flag;
  Buf<long long> uid;
  flag.ensure(nent + 1);
  uid.ensure(nent + 2);
  if (nent > 0) k2_flag<<<nb(nent, 256), 256, 0, st>>>(nent, skeys.p, flag.p);
  xscan(flag.p, uid.p, nent, st, tmp);
  const long long nu = read1(uid.p + nent, st);
  ukeys.ensure(nu + 1);
  uvals.ensure(nu + 1);
  if (nent > 0)
    k2_segsum<<<nb(nent, 256), 256, 0, st>>>(nent, skeys.p, svals.p, flag.p, uid.p, ukeys.p,
                                             uvals.p);
  CK2(cudaEventRecord(ep[2], st));
  // CSR: mirror the upper triangle, sort by (row, col), count rows
  const int U = D.U;
  Buf<double> rhs, fv, fv2;
  Buf<unsigned long long> fk, fk2;
  Buf<int> fflag, rowcnt, col;
  rhs.ensure(U + 1);
  CK2(cudaMemsetAsync(rhs.p, 0, (U + 1) * sizeof(double), st));
  fk.ensure(2 * nu + 1);
  fv.ensure(2 * nu + 1);
  fflag.ensure(2 * nu + 1);
  if (nu > 0) k2_mirror<<<nb(nu, 256), 256, 0, st>>>(nu, ukeys.p, uvals.p, fk.p, fv.p, fflag.p, rhs.p);
  fk2.ensure(2 * nu + 1);
  fv2.ensure(2 * nu + 1);
  if (nu > 0) {
    size_t bytes = 0;
    CK2(cub::DeviceRadixSort::SortPairs(nullptr, bytes, fk.p, fk2.p, fv.p, fv2.p, 2 * nu, 0,
                                        key_bits, st));
    tmp.ensure(bytes);
    CK2(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, fk.p, fk2.p, fv.p, fv2.p, 2 * nu, 0,
                                        key_bits, st));
  }
  Buf<long long> nnzc;
  nnzc.ensure(2 * nu + 2);
  xscan(fflag.p, nnzc.p, 2 * nu, st, tmp);
  const long long nnz = read1(nnzc.p + 2 * nu, st);
  rowcnt.ensure(U + 1);
  CK2(cudaMemsetAsync(rowcnt.p, 0, (U + 1) * sizeof(int), st));
  col.ensure(nnz + 1);
  Buf<double> val;
  val.ensure(nnz + 1);
  if (nnz > 0) k2_csr<<<nb(nnz, 256), 256, 0, st>>>(nnz, fk2.p, fv2.p, rowcnt.p, col.p, val.p);
  Buf<long long> rp;
  rp.ensure(U + 1);
  xscan(rowcnt.p, rp.p, U, st, tmp);
  CK2(cudaEventRecord(e1, st));
  CK2(cudaGetLastError());
  // results
  if (nnz > 2147483647LL) throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: nnz exceeds int32 CSR"};
  out->rows = U;
  out->nnz = nnz;
  out->row_ptr = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (U + 1)));
  out->col_idx = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<long long>(nnz, 1)));
  out->values = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(nnz, 1)));
  out->rhs = static_cast<double*>(std::malloc(sizeof(double) * std::max(U, 1)));
  if (!out->row_ptr || !out->col_idx || !out->values || !out->rhs)
    throw Fail2{NLFEM_GPU_ENOMEM, "out of host memory"};
  std::vector<long long> rph(U + 1);
  CK2(cudaMemcpyAsync(rph.data(), rp.p, sizeof(long long) * (U + 1), cudaMemcpyDeviceToHost, st));
  if (nnz) {
    CK2(cudaMemcpyAsync(out->col_idx, col.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
    CK2(cudaMemcpyAsync(out->values, val.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
  }
  if (U) CK2(cudaMemcpyAsync(out->rhs, rhs.p, sizeof(double) * U, cudaMemcpyDeviceToHost, st));
  unsigned long long c[4];
  CK2(cudaMemcpyAsync(c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost, st));
  CK2(cudaStreamSynchronize(st));
  for (int i = 0; i <= U; ++i) out->row_ptr[i] = (int32_t)rph[i];
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    float ms = 0;
    CK2(cudaEventElapsedTime(&ms, e0, e1));
    stats->device_ms = ms;
    // phases: grid + pairs, integration (entries), sort + segmented sums, CSR
    cudaEvent_t seq[5] = {e0, ep[0], ep[1], ep[2], e1};
    for (int i = 0; i < 4; ++i) {
      CK2(cudaEventElapsedTime(&ms, seq[i], seq[i + 1]));
      stats->phase_ms[i] = ms;
    }
    stats->threads = 1;
    stats->blocks = (KI + 31) / 32;
    stats->mc_samples = c[0];
    stats->mc_hits = c[1];
    stats->items = (long long)c[2];
    stats->element_pairs = npairs;
    stats->shard_pairs = npairs;
    stats->nnz_ext = nnz;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  }
}

}  // namespace

extern "C" int nlfem_gpu_assemble_2d(const nlfem_gpu_mesh2d* mesh, const nlfem_gpu_dofs* dofs,
                                     const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                                     const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                                     nlfem_gpu_csr* out, nlfem_gpu_stats* stats, char* err,
                                     size_t errlen) {
  auto put = [&](const std::string& msg) {
    if (err && errlen) {
      std::strncpy(err, msg.c_str(), errlen - 1);
      err[errlen - 1] = 0;
    }
  };
  try {
    if (!mesh || !dofs || !kernel || !f || !g || !cfg || !out)
      throw Fail2{NLFEM_GPU_BAD_CONFIG, "BadConfig: null argument"};
    out->row_ptr = out->col_idx = nullptr;
    out->values = out->rhs = nullptr;
    assemble2d(mesh, dofs, kernel, f, g, cfg, out, stats);
    return 0;
  } catch (const Fail2& e) {
    put(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    put(e.what());
    return NLFEM_GPU_ENODEVICE;
  }
}
