// nlfem_gpu.cu -- B200 (sm_100a) nonlocal stiffness assembly behind the C-ABI
// declared in include/nlfem_gpu.h.  Drop-in for nlfem::assemble
// (reference proj/src/assembly.cpp:617-843) for the barycenter, nocaps and
// fullcaps strategies.
//
// Pipeline (one CUDA stream, DESIGN.md has the roofline of each stage):
//   prep      element records (128 B/elem), uniform grid over element centers,
//             node->element incidence, per-row fixed-point scales
//   K1 pairs  warp per outer element T: grid candidates, the reference's exact
//             per-(T,q,T') predicates -> element-pair list with 5-bit class
//             codes per quadrature point (two passes: count, fill)
//   K5 pattern node rows R(i) = nodes of partners of T ∋ i, S = R ∪ R^T,
//             mirror slots, element edge slots, unknown-only output CSR
//   K3/K4     CTA per outer element: closed-form whole elements, Gauss on
//             straddle sub-simplices (thread per pair), Philox Monte Carlo caps
//             (warp per cap item) -> 4x4 element-pair blocks, scattered as
//             exact int64 fixed point into the node pattern
//   K6        fixed point -> FP64, mirror, constraint folding into the rhs
//
// Determinism: every value that reaches the matrix is a deterministic FP64
// number converted to int64 with a power-of-two per-row scale; integer adds
// are associative, so the result is bitwise identical for any launch order,
// block count or GPU count.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "geom.cuh"
#include "nlfem_gpu.h"
#include "nlfem_mc_stream.h"

#define FULLMASK 0xffffffffu

namespace {

// ---------------------------------------------------------------------------
// error plumbing

struct Fail {
  int code;
  std::string msg;
};

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw Fail{NLFEM_GPU_ENODEVICE, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

void put_err(char* err, size_t len, const std::string& m) {
  if (!err || len == 0) return;
  std::strncpy(err, m.c_str(), len - 1);
  err[len - 1] = 0;
}

// ---------------------------------------------------------------------------
// device parameter block

constexpr int kMaxTerms = 32;

struct Poly {
  int n;
  double c[kMaxTerms];
  int e[kMaxTerms][3];
};

__device__ __forceinline__ double poly_eval(const Poly& P, Vd p) {
  // Polynomial::eval (reference polynomial.cpp:28-37)
  double acc = 0;
  // the same multiplications in the same order, with short exponents unrolled
  // (data-dependent loops cost more than the arithmetic)
  auto powmul = [](double v, double x, int e) {
    switch (e) {
      case 0: return v;
      case 1: return v * x;
      case 2: return (v * x) * x;
      case 3: return ((v * x) * x) * x;
      default:
        for (int i = 0; i < e; ++i) v *= x;
        return v;
    }
  };
  for (int t = 0; t < P.n; ++t) {
    double v = P.c[t];
    v = powmul(v, p.x, P.e[t][0]);
    v = powmul(v, p.y, P.e[t][1]);
    v = powmul(v, p.z, P.e[t][2]);
    acc += v;
  }
  return acc;
}

struct Dev {
  int K, J, KI, unknowns;
  int strategy, mc;
  unsigned long long seed;
  uint32_t rkey[20];  // Philox round keys (k0 + r W0, k1 + r W1), r < NLFEM_MC_ROUNDS
  double inv_mc;      // 1 / mc when mc is a power of two (vol * inv_mc == vol / mc), else 0
  double C, delta, slack, inside_cut, dd;
  // element data
  const double4* erec;  // [4K]: (c, r), (v0, v1.x), (v1.yz, v2.xy), (v2.z, v3)
  const double* gbar;   // [K] constraint elements: sum_k vol/4 g(x_k) (whole-element Sg)
  const double* cert2;  // [K] nocaps certificate threshold (cert_threshold2)
  const unsigned char* bnd;  // [K] 1 if the element has an unglued facet
  const int4* verts;
  const int4* nbr;
  const double* vol;
  const double* tau;
  const double* diam;
  const double* inv;  // [9K]
  const uint8_t* region;
  const int* interior;  // [KI]
  const int* ipos;      // [K] element -> position in interior[] (-1: constraint)
  const int* dof;       // [J]
  const double* node;   // [3J]
  // grid
  double gox, goy, goz, ginv, hg, rmax;
  int gx, gy, gz;
  const int* cell_start;
  const int* cell_elems;
  const double4* cell_cen;  // [K] (center, radius) of cell_elems[k]: the K1 screen reads
                            // it coalesced, beside the id instead of after it
  // node incidence (interior elements) sorted by element id
  const int* ni_off;
  const int* ni_el;
  // fixed point
  const double* scale;
  const double* iscale;
  const double4* escale;      // [K] fixed-point scales of the element's 4 nodes
  const unsigned char* econ;  // [K] bit k: node k of the element is constrained
  Poly f, g;
  unsigned long long* flags;  // counter 7: approxcaps hull face-table overflow
};

__constant__ Dev cD;

__device__ __forceinline__ void load_elem(int t, Vd& c, double& r, Vd v[4]) {
  const double4 a = cD.erec[4 * t], b = cD.erec[4 * t + 1], e = cD.erec[4 * t + 2],
                d = cD.erec[4 * t + 3];
  c = {a.x, a.y, a.z};
  r = a.w;
  v[0] = {b.x, b.y, b.z};
  v[1] = {b.w, e.x, e.y};
  v[2] = {e.z, e.w, d.x};
  v[3] = {d.y, d.z, d.w};
}

__device__ __forceinline__ void load_verts(int t, Vd v[4]) {
  const double4 b = cD.erec[4 * t + 1], e = cD.erec[4 * t + 2], d = cD.erec[4 * t + 3];
  v[0] = {b.x, b.y, b.z};
  v[1] = {b.w, e.x, e.y};
  v[2] = {e.z, e.w, d.x};
  v[3] = {d.y, d.z, d.w};
}

// ---------------------------------------------------------------------------
// generic helpers: exclusive scan of int64 counts (3-phase, deterministic)

constexpr int kScanBlock = 1024;

template <class Tin>
__global__ void k_scan_block(const Tin* in, long long* out, long long* sums, long long n) {
  __shared__ long long s[kScanBlock];
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  s[threadIdx.x] = i < n ? (long long)in[i] : 0;
  __syncthreads();
  for (int off = 1; off < kScanBlock; off <<= 1) {
    long long v = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  if (i < n) out[i] = s[threadIdx.x] - (i < n ? (long long)in[i] : 0);
  if (threadIdx.x == kScanBlock - 1) sums[blockIdx.x] = s[threadIdx.x];
}

// single-CTA exclusive scan for small n (one launch, total written to out[n]):
// thread t scans its contiguous slice, warp and block prefixes of the slice sums
constexpr int kScan1Threads = 1024;
constexpr long long kScan1Max = 64 * 1024;
template <class Tin>
__global__ void __launch_bounds__(kScan1Threads) k_scan_one(const Tin* in, long long* out,
                                                            long long n) {
  __shared__ long long wsum[kScan1Threads / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const long long per = (n + kScan1Threads - 1) / kScan1Threads;
  const long long lo = min(n, (long long)t * per), hi = min(n, lo + per);
  long long acc = 0;
  for (long long i = lo; i < hi; ++i) acc += (long long)in[i];
  long long inc = acc;
  for (int sh = 1; sh < 32; sh <<= 1) {
    const long long y = __shfl_up_sync(FULLMASK, inc, sh);
    if (lane >= sh) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  long long wbase = 0, total = 0;
  for (int w = 0; w < kScan1Threads / 32; ++w) {
    wbase += w < wid ? wsum[w] : 0;
    total += wsum[w];
  }
  long long run = wbase + inc - acc;
  for (long long i = lo; i < hi; ++i) {
    const long long v = (long long)in[i];
    out[i] = run;
    run += v;
  }
  if (t == 0) out[n] = total;
}

__global__ void k_scan_add(long long* out, const long long* offs, long long n) {
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += offs[blockIdx.x];
}

// ---------------------------------------------------------------------------
// prep kernels


__device__ __forceinline__ int cell_of(double c, double o, double inv, int n) {
  int k = (int)floor((c - o) * inv);
  return k < 0 ? 0 : (k >= n ? n - 1 : k);
}


__global__ void k_fill_by_key(int n, const int* key, const long long* off, int* cursor, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int k = key[t];
  const int pos = atomicAdd(cursor + k, 1);
  out[off[k] + pos] = t;
}

// Sort each short segment ascending (insertion sort, one thread per segment);
// makes the atomic fills deterministic.
__global__ void k_cell_cen(int K, const int* cell_elems, const double4* erec, double4* cen) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K) cen[k] = erec[4 * (long long)cell_elems[k]];
}

__global__ void k_sort_segments(int nseg, const long long* off, int* data) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const long long a = off[s], b = off[s + 1];
  for (long long i = a + 1; i < b; ++i) {
    const int x = data[i];
    long long j = i - 1;
    while (j >= a && data[j] > x) {
      data[j + 1] = data[j];
      --j;
    }
    data[j + 1] = x;
  }
}

// node -> interior-element incidence (count / fill by (node, elem) items)

__global__ void k_ninc_fill(int K, const long long* off, int* cursor, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K || cD.region[t]) return;
  const int4 w = cD.verts[t];
  const int v[4] = {w.x, w.y, w.z, w.w};
  for (int i = 0; i < 4; ++i) out[off[v[i]] + atomicAdd(cursor + v[i], 1)] = t;
}

// per-node patch volume over all elements -> power-of-two fixed-point scale
// per row: bound of every contribution (count x largest incident volume, an
// upper bound of the patch volume that is independent of summation order)
__global__ void k_scales(int J, const int* acnt, const unsigned long long* avmax, double cbound,
                         double* scale, double* iscale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= J) return;
  const double patch = (double)acnt[i] * __longlong_as_double((long long)avmax[i]);
  const double bound = cbound * (patch > 0 ? patch : 1e-300);
  int ex;
  frexp(bound, &ex);  // bound < 2^ex
  scale[i] = ldexp(1.0, 61 - ex);
  iscale[i] = ldexp(1.0, ex - 61);
}



// ---------------------------------------------------------------------------
// per element: the scales and constrained flags of its four nodes, so the
// combine reads them with the partner id (one gather level instead of two)
__global__ void k_elem_scales(int K, const double* scale, double4* escale, unsigned char* econ) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const int4 w = cD.verts[t];
  escale[t] = make_double4(scale[w.x], scale[w.y], scale[w.z], scale[w.w]);
  econ[t] = (unsigned char)((cD.dof[w.x] < 0) | ((cD.dof[w.y] < 0) << 1) |
                            ((cD.dof[w.z] < 0) << 2) | ((cD.dof[w.w] < 0) << 3));
}

// K1: element pairs

// Class codes (5 bits per quadrature point): 0 none, 1 whole element,
// 2 Monte Carlo cap over the whole element (fullcaps, all vertices outside),
// 16|mask straddling element with inside-vertex mask 1..14.
enum : unsigned { kNone = 0, kWhole = 1, kOutCap = 2, kStraddle = 16 };

__device__ __forceinline__ int count_kept(const Straddle& st, double tau) {
  int n = 0;
  for (int k = 0; k < st.n; ++k) {
    Vd a, b, c, d;
    straddle_piece(st, k, a, b, c, d);
    n += tet_volume(a, b, c, d) > tau;
  }
  return n;
}

// Exact piece tests: does straddle_inner (nocaps) or straddle_inner +
// straddle_outer (fullcaps) keep at least one sub-simplex above the volume floor?
__device__ __noinline__ bool inner_pieces_exact(const Vd* v, int mask, Vd xq, double tau) {
  return count_kept(inner_straddle(v, mask, xq, cD.delta), tau) > 0;
}

__device__ __noinline__ bool any_pieces_exact(const Vd* v, int mask, Vd xq, double tau) {
  return count_kept(inner_straddle(v, mask, xq, cD.delta), tau) +
             count_kept(outer_straddle(v, mask, xq, cD.delta), tau) > 0;
}

// approxcaps: does the sphere-point hull keep a fan piece above the floor?
// (a face-table overflow -- impossible for <= 10 points -- is flagged in
// counter 7 and fails the run)
__device__ __noinline__ bool approx_pieces_exact(const Vd* v, int mask, Vd xq, double tau) {
  int kept = 0;
  const bool ok = approx_pieces(v, mask, xq, cD.delta, tau,
                                [&](Vd, Vd, Vd, Vd, double) { ++kept; });
  if (!ok) atomicOr(cD.flags, 1ull);
  return kept > 0;
}

// Nocaps certificate (used by classify_cheap): the inner polytope contains a
// tet of volume >= (depth/diam)^(4-m) vol(T'), depth = delta - |v - x_q| of the
// deepest inside vertex, and its <= 3 kept pieces tile the polytope, so some
// piece exceeds tau once depth > rho = diam * max((8 tau / vol)^(1/3), 1e-6)
// (the largest of the m-wise thresholds).  Tested on squared distances with a
// factor-2 margin; otherwise the exact decomposition decides.
__device__ __forceinline__ double cert_threshold2(double diam, double vol, double tau) {
  const double rho = diam * fmax(cbrt(8.0 * tau / vol), 1e-6);
  const double t = cD.delta - 2.0 * rho;
  return t > 0 ? t * t * (1.0 - 1e-12) : 0.0;
}

// Element-wise preparation in one pass: the 128-byte element record, the
// whole-constraint g average, the nocaps certificate and unglued-facet flag,
// the grid cell (key and count), and per node the number of interior and of
// all incident elements and the largest incident volume (row bounds).
__global__ void k_elem_prep(int K, const double* node, const int4* verts, const double* center,
                            const double* radius, double4* erec, double* gbar, double* cert2,
                            unsigned char* bnd, int* cell_key, int* cell_cnt, int* ni_cnt,
                            int* ai_cnt, unsigned long long* ai_vmax) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const int4 w = verts[t];
  const double* a = node + 3 * (long long)w.x;
  const double* b = node + 3 * (long long)w.y;
  const double* c = node + 3 * (long long)w.z;
  const double* d = node + 3 * (long long)w.w;
  const double cx = center[3 * t], cy = center[3 * t + 1], cz = center[3 * t + 2];
  erec[4 * t] = make_double4(cx, cy, cz, radius[t]);
  erec[4 * t + 1] = make_double4(a[0], a[1], a[2], b[0]);
  erec[4 * t + 2] = make_double4(b[1], b[2], c[0], c[1]);
  erec[4 * t + 3] = make_double4(c[2], d[0], d[1], d[2]);
  const double vol = cD.vol[t];
  const bool interior = cD.region[t] == 0;
  double Sg = 0;
  if (!interior) {  // whole constraint element (reference assembly.cpp:350-359)
    const Vd v[4] = {{a[0], a[1], a[2]}, {b[0], b[1], b[2]}, {c[0], c[1], c[2]}, {d[0], d[1], d[2]}};
    for (int k = 0; k < 4; ++k) Sg += vol * 0.25 * poly_eval(cD.g, quad_point(v, k));
  }
  gbar[t] = Sg;
  cert2[t] = cert_threshold2(cD.diam[t], vol, cD.tau[t]);
  const int4 nb = cD.nbr[t];
  bnd[t] = (nb.x < 0 || nb.y < 0 || nb.z < 0 || nb.w < 0) ? 1 : 0;
  const int kx = cell_of(cx, cD.gox, cD.ginv, cD.gx);
  const int ky = cell_of(cy, cD.goy, cD.ginv, cD.gy);
  const int kz = cell_of(cz, cD.goz, cD.ginv, cD.gz);
  const int key = (kz * cD.gy + ky) * cD.gx + kx;
  cell_key[t] = key;
  atomicAdd(cell_cnt + key, 1);
  const int vv[4] = {w.x, w.y, w.z, w.w};
  const unsigned long long vb = (unsigned long long)__double_as_longlong(vol);  // vol > 0
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (interior) atomicAdd(ni_cnt + vv[k], 1);
    atomicAdd(ai_cnt + vv[k], 1);
    atomicMax(ai_vmax + vv[k], vb);
  }
}

// distance_point_simplex(xq, v) < delta, decided from the facets that can hold
// the closest point: for xq outside T' the closest point lies on a facet whose
// plane separates xq (lambda_f < 0), so the minimum over facets with
// lambda_f < 1e-6 (a margin far above rounding) is the true distance up to
// rounding.  Conclusive when it is 1e-9 delta away from delta; otherwise the
// reference expression decides.
__device__ __noinline__ bool outside_cap_hits(Vd xq, const Vd* v, double delta) {
  const Vd e1 = vsub(v[1], v[0]), e2 = vsub(v[2], v[0]), e3 = vsub(v[3], v[0]);
  const Vd b = vsub(xq, v[0]);
  const double det = vdot(e1, vcross(e2, e3));
  const double l1 = vdot(b, vcross(e2, e3)) / det;
  const double l2 = vdot(e1, vcross(b, e3)) / det;
  const double l3 = vdot(e1, vcross(e2, b)) / det;
  const double l0 = 1.0 - l1 - l2 - l3;
  if (!(l0 < 0) && !(l1 < 0) && !(l2 < 0) && !(l3 < 0)) return true;  // inside: 0 < delta
  const double lam[4] = {l0, l1, l2, l3};
  double d = INFINITY;
  for (int f = 0; f < 4; ++f)
    if (lam[f] < 1e-6) d = fmin(d, facet_distance(v, f, xq));
  if (d < delta * (1.0 - 1e-9)) return true;
  if (d > delta * (1.0 + 1e-9)) return false;
  return distance_point_simplex(xq, v) < delta;
}

// BallExitsMesh probe: an unglued facet of T' closer than delta - slack to xq.
// The facet's plane distance bounds its triangle distance from below; facets
// whose plane is farther than the threshold (1e-9 relative margin) are skipped.
__device__ __noinline__ bool facet_too_close(const Vd* v, int4 nb, Vd xq) {
  const int nbv[4] = {nb.x, nb.y, nb.z, nb.w};
  const double thr = cD.delta - cD.slack;
  for (int f = 0; f < 4; ++f) {
    if (nbv[f] >= 0) continue;
    const Vd a = v[f == 0 ? 1 : 0], bb = v[f <= 1 ? 2 : 1], c = v[f <= 2 ? 3 : 2];
    const Vd n = vcross(vsub(bb, a), vsub(c, a));
    const double h = vdot(n, vsub(xq, a));
    if (h * h > thr * thr * vnorm2(n) * (1.0 + 1e-9)) continue;
    if (facet_distance(v, f, xq) < thr) return true;
  }
  return false;
}

// The reference's per-(T,q,T') decision (assembly.cpp:722-759), split in two:
// classify_cheap settles every item that the screens, certificates and
// classify_simplex decide, and returns kDefer | mask for the few that need an
// exact geometric evaluation (classify_deferred), so a warp can queue those and
// work them with all lanes.
constexpr unsigned kDefer = 0x80u;
// STRAT: the strategy as a compile-time constant (k_pairs is instantiated per
// strategy, so each instance carries only its own decision code)
template <int STRAT>
__device__ __forceinline__ unsigned classify_cheap(Vd xq, Vd cen, double rad, const Vd v[4],
                                                   double cert2, double vol, double tau) {
  const double delta = cD.delta;
  // The reference compares gap = sqrt(|c - x_q|^2) against thresholds.  A
  // squared comparison with a 1e-12 relative margin decides the same way
  // whenever it is conclusive (sqrt and the square are correctly rounded);
  // otherwise fall through to the reference's exact expression.
  const double g2 = vnorm2(vsub(cen, xq));
  const double t1 = rad + delta;
  if (g2 >= t1 * t1 * (1.0 + 1e-12)) return kNone;
  double gap = -1.0;  // computed lazily
  if (!(g2 < t1 * t1 * (1.0 - 1e-12))) {
    gap = sqrt(g2);
    if (gap >= rad + delta) return kNone;
  }
  if (STRAT == NLFEM_STRATEGY_OVERLAP) {
    // gap + rad < delta || distance_point_simplex(x_q, T') < delta
    const double t2 = delta - rad;
    if (t2 > 0) {
      if (g2 < t2 * t2 * (1.0 - 1e-12)) return kWhole;
      if (!(g2 >= t2 * t2 * (1.0 + 1e-12))) {
        if (gap < 0) gap = sqrt(g2);
        if (gap + rad < delta) return kWhole;
      }
    }
    // a point of T' (barycenter or vertex) well inside the ball certifies the
    // computed distance < delta; otherwise evaluate it (classify_deferred)
    const double c2 = delta * delta * (1.0 - 1e-11);
    if (g2 < c2) return kWhole;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (vnorm2(vsub(v[i], xq)) < c2) return kWhole;
    return kDefer;
  }
  if (STRAT == NLFEM_STRATEGY_BARYCENTER) {
    if (g2 < delta * delta * (1.0 - 1e-12)) return kWhole;
    if (g2 >= delta * delta * (1.0 + 1e-12)) return kNone;
    if (gap < 0) gap = sqrt(g2);
    return gap < delta ? kWhole : kNone;
  }
  // fast inside cut: gap + rad < inside_cut
  const double t2 = cD.inside_cut - rad;
  if (t2 > 0) {
    if (g2 < t2 * t2 * (1.0 - 1e-12)) return kWhole;
    if (!(g2 >= t2 * t2 * (1.0 + 1e-12))) {
      if (gap < 0) gap = sqrt(g2);
      if (gap + rad < cD.inside_cut) return kWhole;
    }
  }
  // classify_simplex flags (reference geometry.cpp:8-24), keeping |v - x_q|^2
  double d2[4];
  int mask = 0;
  {
    const double r_in = delta - 1e-10 * delta;
    const double r2 = r_in * r_in;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      d2[i] = vnorm2(vsub(v[i], xq));
      if (d2[i] < r2) mask |= 1 << i;
    }
  }
  if (mask == 15) return kWhole;
  if (STRAT == NLFEM_STRATEGY_INSIDE) return kNone;  // straddlers dropped
  if (mask == 0) {
    if (STRAT != NLFEM_STRATEGY_FULLCAPS) return kNone;
    // the barycenter lies in T': gap < delta (with margin) certifies that the
    // computed distance_point_simplex is < delta; otherwise evaluate it
    if (g2 < delta * delta * (1.0 - 1e-11)) return kOutCap;
    return kDefer;
  }
  if (STRAT == NLFEM_STRATEGY_NOCAPS || STRAT == NLFEM_STRATEGY_APPROXCAPS) {
    // (approxcaps: the hull contains the nocaps polytope, whose certified
    // volume > 64 tau exceeds its <= 16 fan pieces x tau)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((mask >> i & 1) && d2[i] < cert2) return kStraddle | mask;
    return kDefer | mask;
  }
  if (vol > 64.0 * tau) return kStraddle | mask;  // inner + outer polytopes cover T'
  return kDefer | mask;
}

template <int STRAT>
__device__ __forceinline__ unsigned classify_deferred(Vd xq, const Vd v[4], int mask, double tau) {
  if (mask == 0)
    return outside_cap_hits(xq, v, cD.delta)
               ? (STRAT == NLFEM_STRATEGY_OVERLAP ? kWhole : kOutCap)
               : kNone;
  if (STRAT == NLFEM_STRATEGY_NOCAPS)
    return inner_pieces_exact(v, mask, xq, tau) ? (kStraddle | mask) : kNone;
  if (STRAT == NLFEM_STRATEGY_APPROXCAPS)
    return approx_pieces_exact(v, mask, xq, tau) ? (kStraddle | mask) : kNone;
  return any_pieces_exact(v, mask, xq, tau) ? (kStraddle | mask) : kNone;
}

struct OuterT {
  int T;
  Vd c;
  Vd v[4];
  double R;
};

__device__ __forceinline__ void outer_setup(int T, OuterT& o) {
  double r;
  load_elem(T, o.c, r, o.v);
  double spread = 0;
  for (int k = 0; k < 4; ++k) spread = fmax(spread, vdist(quad_point(o.v, k), o.c));
  o.T = T;
  o.R = cD.delta + spread;
}

constexpr int kPairThreads = 128;       // 4 warps = 4 consecutive outer elements
constexpr int kPairWarps = kPairThreads / 32;
constexpr int kCandChunk = 128;         // candidates staged in shared memory at a time

struct CandStage {
  double4 rec[kCandChunk][4];  // erec of the candidate (center+radius, vertices)
  double vol[kCandChunk], tau[kCandChunk], cert2[kCandChunk];
  int id[kCandChunk];
  unsigned char pass[kCandChunk];  // bit w: passes warp w's superset screen
  unsigned char bnd[kCandChunk];   // candidate has an unglued facet
  short mine[kPairWarps][kCandChunk];  // per warp: indices of its candidates
};

// CTA per 4 consecutive outer elements T (one per warp).  The CTA streams the
// grid rows of the union of their reach boxes once; a candidate T' survives if
// its bounding sphere can reach B(delta) of some quadrature point of one of the
// four T (a conservative superset of the reference's BFS superset,
// assembly.cpp:569-613).
//   MODE 0: count each warp's survivors (no classification);
//   MODE 1: stage survivors in shared memory; each warp classifies its own with
//           one lane per (candidate, quadrature point) -- the reference's exact
//           per-(T,q,T') predicates -- ORs the four 5-bit codes and writes
//           (T', code) into its survivor slots (code 0 = no piece), in stream
//           order; k_pairs_compact then keeps the nonzero ones.
//   WIDE: one outer element per CTA, its staged survivors split over the four
//         warps in groups of 8 (small ranges, e.g. one rank's shard: four times
//         the warps per element, a quarter of the per-CTA latency).
template <int MODE, bool WIDE = false, int STRAT = NLFEM_STRATEGY_FULLCAPS>
#ifndef NLFEM_PAIRS_MINBLOCKS
#define NLFEM_PAIRS_MINBLOCKS 6
#endif
__global__ void __launch_bounds__(kPairThreads, NLFEM_PAIRS_MINBLOCKS) k_pairs(int ii_base, int ii_end,
                                                        const long long* cand_off,
                                                        long long cand_base, int* cand_count,
                                                        int* cpartner, unsigned* cinfo,
                                                        int* pair_count,
                                                        unsigned long long* item_count,
                                                        int* err_elem) {
  __shared__ CandStage sg;
  __shared__ int xb[6], scnt[kPairWarps];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  // outer element index
  const int warp = ii_base + (WIDE ? (int)blockIdx.x : (int)blockIdx.x * kPairWarps + wl);
  const bool active = warp < ii_end;
  OuterT o;
  if (active) outer_setup(cD.interior[warp], o);
  else o.R = -1;
  const double reach = o.R + cD.rmax;
  if (threadIdx.x == 0) {
    xb[0] = xb[2] = xb[4] = 1 << 30;
    xb[1] = xb[3] = xb[5] = -1;
  }
  if (threadIdx.x < kPairWarps) scnt[threadIdx.x] = 0;
  __syncthreads();
  if (active && lane == 0) {
    atomicMin(xb + 0, cell_of(o.c.x - reach, cD.gox, cD.ginv, cD.gx));
    atomicMax(xb + 1, cell_of(o.c.x + reach, cD.gox, cD.ginv, cD.gx));
    atomicMin(xb + 2, cell_of(o.c.y - reach, cD.goy, cD.ginv, cD.gy));
    atomicMax(xb + 3, cell_of(o.c.y + reach, cD.goy, cD.ginv, cD.gy));
    atomicMin(xb + 4, cell_of(o.c.z - reach, cD.goz, cD.ginv, cD.gz));
    atomicMax(xb + 5, cell_of(o.c.z + reach, cD.goz, cD.ginv, cD.gz));
  }
  __syncthreads();
  const int x0 = xb[0], x1 = xb[1], y0 = xb[2], y1 = xb[3], z0 = xb[4], z1 = xb[5];
  __shared__ double oc[kPairWarps][4];
  // the outer element's quadrature points, parked in shared memory (the
  // classification reads them; keeping T's vertices live in registers across
  // the candidate stream made ptxas spill)
  __shared__ double oq[kPairWarps][4][3];
  if (lane == 0) {
    oc[wl][0] = o.c.x;
    oc[wl][1] = o.c.y;
    oc[wl][2] = o.c.z;
    oc[wl][3] = active ? o.R : -1.0;
  }
  if (lane < 4) {
    const Vd x = active ? quad_point(o.v, lane) : Vd{0, 0, 0};
    oq[wl][lane][0] = x.x;
    oq[wl][lane][1] = x.y;
    oq[wl][lane][2] = x.z;
  }
  __syncthreads();
  const long long out = (MODE == 1 && active) ? cand_off[warp] - cand_base : 0;
  int cnt = 0, npair = 0;
  unsigned items = 0;

  // per warp: the 4 x 5-bit code of each of its candidates, and the queue of
  // deferred items (bits 0-3 mask, 4 classify, 5 facet probe, 6-7 q, 8-14 index)
  __shared__ unsigned wcode[kPairWarps][kCandChunk];
  __shared__ unsigned short wdef[kPairWarps][4 * kCandChunk];
  int nreg = 0;  // candidates staged so far (same value in every thread)
  auto classify_chunk = [&]() {
    int nm = 0;
    for (int base = 0; base < nreg; base += 32) {
      const int k = base + lane;
      const bool mine =
          k < nreg && (WIDE ? (((k >> 3) & (kPairWarps - 1)) == wl) : ((sg.pass[k] >> wl) & 1));
      const unsigned bal = __ballot_sync(FULLMASK, mine);
      if (mine) sg.mine[wl][nm + __popc(bal & ((1u << lane) - 1))] = (short)k;
      nm += __popc(bal);
    }
    __syncwarp();
    // pass 1: lane = (candidate, quadrature point), cheap decisions
    int nd = 0;
    for (int base = 0; base < nm; base += 8) {
      const int t = base + (lane >> 2), q = lane & 3;
      unsigned code = 0, ent = 0;
      if (t < nm) {
        const int k = sg.mine[wl][t];
        const double4 a = sg.rec[k][0], b = sg.rec[k][1], e = sg.rec[k][2], d = sg.rec[k][3];
        const Vd cp = {a.x, a.y, a.z};
        const Vd v[4] = {{b.x, b.y, b.z}, {b.w, e.x, e.y}, {e.z, e.w, d.x}, {d.y, d.z, d.w}};
        const Vd xq = {oq[wl][q][0], oq[wl][q][1], oq[wl][q][2]};
        const unsigned c =
            classify_cheap<STRAT>(xq, cp, a.w, v, sg.cert2[k], sg.vol[k], sg.tau[k]);
        if (c & kDefer) ent = 16u | (c & 15u);
        else code = c << (5 * q);
        if (sg.bnd[k]) ent |= 32u;
        if (ent) ent |= ((unsigned)q << 6) | ((unsigned)t << 8);
      }
      code |= __shfl_xor_sync(FULLMASK, code, 1);
      code |= __shfl_xor_sync(FULLMASK, code, 2);
      if ((lane & 3) == 0 && t < nm) wcode[wl][t] = code;
      const unsigned bal = __ballot_sync(FULLMASK, ent != 0);
      if (ent) wdef[wl][nd + __popc(bal & ((1u << lane) - 1))] = (unsigned short)ent;
      nd += __popc(bal);
    }
    __syncwarp();
    // pass 2: the deferred items, all lanes busy
    for (int i = lane; i < nd; i += 32) {
      const unsigned ent = wdef[wl][i];
      const int t = (int)(ent >> 8), q = (int)((ent >> 6) & 3);
      const int k = sg.mine[wl][t];
      const double4 b = sg.rec[k][1], e = sg.rec[k][2], d = sg.rec[k][3];
      const Vd v[4] = {{b.x, b.y, b.z}, {b.w, e.x, e.y}, {e.z, e.w, d.x}, {d.y, d.z, d.w}};
      const Vd xq = {oq[wl][q][0], oq[wl][q][1], oq[wl][q][2]};
      if (ent & 16u) {
        const unsigned c = classify_deferred<STRAT>(xq, v, (int)(ent & 15u), sg.tau[k]);
        if (c) atomicOr(&wcode[wl][t], c << (5 * q));
      }
      if (ent & 32u) {
        const int Tp = sg.id[k];
        if (facet_too_close(v, cD.nbr[Tp], xq)) atomicMin(err_elem, Tp);
      }
    }
    __syncwarp();
    // write (T', code) into the survivor slots, in stream order
    for (int t = lane; t < nm; t += 32) {
      const unsigned code = wcode[wl][t];
      // survivor slot: the warp's t-th, or (WIDE) the element's staged index
      const long long slot = out + cnt + (WIDE ? sg.mine[wl][t] : t);
      cpartner[slot] = sg.id[sg.mine[wl][t]];
      cinfo[slot] = code;
#pragma unroll
      for (int q = 0; q < 4; ++q) items += ((code >> (5 * q)) & 31u) != 0;
      npair += code != 0;
    }
    __syncwarp();
    cnt += WIDE ? nreg : nm;
  };

  // staging: one block barrier per batch of kPairThreads candidates.  The
  // per-warp survivor counts are double-buffered by batch parity; every thread
  // derives the warp bases and the running staged count itself; the next
  // batch's barrier orders this batch's staging writes before any reads.
  __shared__ int wcount[2][kPairWarps];
  int par = 0;
  // the grid rows of the reach box (z-major, then y; each row a contiguous run
  // of cells x0..x1, hence of cell_elems) are streamed as one flat candidate
  // sequence, a group of rows at a time: batches span row boundaries, so all
  // threads stage a candidate in every batch (same candidate order as a
  // row-by-row walk)
  constexpr int kRowGroup = 256;
  __shared__ int rstart[kRowGroup], rpre[kRowGroup + 1];
  const int ny = y1 - y0 + 1, nz = z1 - z0 + 1;
  const int nrows = (ny > 0 && nz > 0 && x1 >= x0) ? ny * nz : 0;
  for (int rg = 0; rg < nrows; rg += kRowGroup) {
    const int nr = min(kRowGroup, nrows - rg);
    __syncthreads();  // the previous group's row table is no longer read
    for (int t = threadIdx.x; t < nr; t += kPairThreads) {
      const int r = rg + t, z = z0 + r / ny, y = y0 + r % ny;
      const int row = (z * cD.gy + y) * cD.gx;
      const int e0 = cD.cell_start[row + x0], e1 = cD.cell_start[row + x1 + 1];
      rstart[t] = e0;
      rpre[t + 1] = e1 - e0;
    }
    __syncthreads();
    if (wl == 0) {  // inclusive scan of the row lengths
      int carry = 0;
      for (int t0 = 0; t0 < nr; t0 += 32) {
        int v = (t0 + lane < nr) ? rpre[t0 + lane + 1] : 0;
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int u = __shfl_up_sync(FULLMASK, v, sh);
          if (lane >= sh) v += u;
        }
        if (t0 + lane < nr) rpre[t0 + lane + 1] = v + carry;
        carry += __shfl_sync(FULLMASK, v, 31);
      }
      if (lane == 0) rpre[0] = 0;
    }
    __syncthreads();
    const int total = rpre[nr];
    int rr = 0;  // this thread's row (its candidate index only grows)
    {
      for (int base = 0; base < total; base += kPairThreads) {
        const int g = base + threadIdx.x;
        unsigned pm = 0;
        int Tp = -1;
        double4 a;
        if (g < total) {
          while (rpre[rr + 1] <= g) ++rr;
          const int ci = rstart[rr] + (g - rpre[rr]);
          Tp = cD.cell_elems[ci];
          a = cD.cell_cen[ci];
#pragma unroll
          for (int w = 0; w < kPairWarps; ++w) {
            const double thr = a.w + oc[w][3];
            const double dx = a.x - oc[w][0], dy = a.y - oc[w][1], dz = a.z - oc[w][2];
            if (oc[w][3] >= 0 && dx * dx + dy * dy + dz * dz < thr * thr * (1.0 + 1e-10))
              pm |= 1u << w;
          }
        }
        if constexpr (MODE == 0) {
#pragma unroll
          for (int w = 0; w < kPairWarps; ++w) {
            const int c = __popc(__ballot_sync(FULLMASK, (pm >> w) & 1));
            if (lane == 0 && c) atomicAdd(scnt + w, c);
          }
          continue;
        }
        // stage survivors (block-wide compaction, stream order)
        const unsigned bal = __ballot_sync(FULLMASK, pm != 0);
        if (lane == 0) wcount[par][wl] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kPairWarps; ++w) {
          const int c = wcount[par][w];
          before += w < wl ? c : 0;
          tot += c;
        }
        par ^= 1;
        if (nreg + tot > kCandChunk) {
          classify_chunk();
          __syncthreads();  // every warp is done reading the staged chunk
          nreg = 0;
        }
        if (pm) {
          const int k = nreg + before + __popc(bal & ((1u << lane) - 1));
          sg.id[k] = Tp;
          sg.rec[k][0] = a;
          sg.rec[k][1] = cD.erec[4 * Tp + 1];
          sg.rec[k][2] = cD.erec[4 * Tp + 2];
          sg.rec[k][3] = cD.erec[4 * Tp + 3];
          sg.vol[k] = cD.vol[Tp];
          sg.tau[k] = cD.tau[Tp];
          sg.cert2[k] = cD.cert2[Tp];
          sg.bnd[k] = cD.bnd[Tp];
          sg.pass[k] = (unsigned char)pm;
        }
        nreg += tot;
      }
    }
  }
  if (MODE == 0) {
    __syncthreads();
    if (active && lane == 0 && (!WIDE || wl == 0)) cand_count[warp] = scnt[wl];
    return;
  }
  __syncthreads();  // the last batch's staging before the final chunk
  classify_chunk();
  for (int sh = 16; sh > 0; sh >>= 1) {
    items += __shfl_xor_sync(FULLMASK, items, sh);
    npair += __shfl_xor_sync(FULLMASK, npair, sh);
  }
  if (WIDE) {  // the element's pair count over its four warps
    __shared__ int spair;
    if (threadIdx.x == 0) spair = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&spair, npair);
    __syncthreads();
    if (active && threadIdx.x == 0) pair_count[warp] = spair;
    if (active && lane == 0) atomicAdd(item_count, (unsigned long long)items);
    return;
  }
  if (active && lane == 0) {
    pair_count[warp] = npair;
    atomicAdd(item_count, (unsigned long long)items);
  }
}

// keep the survivors with a nonzero code, in order: warp per outer element
__global__ void k_pairs_compact(int ii0, int ii1, const long long* cand_off, long long cand_base,
                                const int* cpartner, const unsigned* cinfo,
                                const long long* pair_off, int* partner, unsigned* info) {
  const int ii = ii0 + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (ii >= ii1) return;
  const long long a = cand_off[ii] - cand_base, b = cand_off[ii + 1] - cand_base;
  long long o = pair_off[ii];
  for (long long k = a; k < b; k += 32) {
    const long long j = k + lane;
    const unsigned c = j < b ? cinfo[j] : 0;
    const unsigned bal = __ballot_sync(FULLMASK, c != 0);
    if (c) {
      const long long pos = o + __popc(bal & ((1u << lane) - 1));
      partner[pos] = cpartner[j];
      info[pos] = c;
    }
    o += __popc(bal);
  }
}

// ---------------------------------------------------------------------------
// K5: pattern

// Pattern tables per node block, in shared memory: element hash slots, node
// hash slots and the longest row.  The small set covers delta/h <~ 5 (row
// lengths ~(4/3) pi (delta/h + 2)^3 nodes); a pass that overflows it is rerun
// with the large set (192 KB of shared memory per block: delta/h <~ 8.5, e.g.
// the finest level of the reference's default convergence study).
struct PatTabs {
  int he, hn, rowmax;
};
constexpr PatTabs kPatSmall{8192, 4096, 4096};
constexpr PatTabs kPatBig{32768, 8192, 8192};

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// insert key into an open-addressing table of ints (-1 = empty); returns true
// when newly inserted, sets *ovf when full.
__device__ __forceinline__ bool hset_insert(int* tab, int cap, int key, int* ovf) {
  unsigned h = hash32((unsigned)key) & (cap - 1);
  for (int probe = 0; probe < cap; ++probe) {
    const int prev = atomicCAS(tab + h, -1, key);
    if (prev == -1) return true;
    if (prev == key) return false;
    h = (h + 1) & (cap - 1);
  }
  *ovf = 1;
  return false;
}

// block-wide bitonic sort of n <= kRowMax ints in shared memory (ascending)
__device__ void block_sort(int* a, int n) {
  int p = 1;
  while (p < n) p <<= 1;
  for (int i = n + threadIdx.x; i < p; i += blockDim.x) a[i] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= p; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < p; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const int x = a[i], y = a[ixj];
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Pattern pass with speculative capacities: a size-dependent kernel does nothing
// once a total has exceeded its buffer (ovf = kCapRetry; the host then reruns
// the pass with exact sizes), or once an error has been flagged.
constexpr int kCapRetry = 9;
__global__ void k_cap_check(const long long* total, long long cap, int* ovf) {
  if (threadIdx.x == 0 && *total > cap) atomicCAS(ovf, 0, kCapRetry);
}

// R(i) = sorted nodes of interior partners of every interior T containing node i.
// flag the interior partners of a pair range (pairs [0, *pend))
__global__ void k_mark_partners(long long np, const long long* pend, const int* partner,
                                unsigned char* mark) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np || p >= *pend) return;
  const int Tp = partner[p];
  if (cD.region[Tp] == 0) mark[Tp] = 1;
}

// plo / phi: the outer elements (interior positions) whose pairs are built
// (the whole interior list on one GPU; a rank's range under the owner-computes
// multi-GPU plan); pmark (or null): interior elements that
// are partners of those pairs -- their own node pairs enter the rows too, so a
// rank's local pattern holds every slot its combine adds to (the D_T' block)
// MODE 0: row lengths; 1: rows written at roff (from the scanned lengths);
// 2: one pass -- each row takes its place in rcols from a global cursor (rows in
// arrival order: roff[i] = its start, rlen[i] = its length, roff[J] = the total;
// the row contents, hence everything derived from them, do not depend on the
// order), nothing written once the cursor passes cap (ovf = kCapRetry).
template <int MODE>
__global__ void __launch_bounds__(256) k_rows(const long long* pair_off, const int* partner,
                                              int* rlen, long long* roff, int* rcols,
                                              int* ovf, int plo, int phi,
                                              const unsigned char* pmark, PatTabs tb,
                                              unsigned long long* cursor, long long cap) {
  constexpr bool FILL = MODE != 0;
  extern __shared__ int sm[];
  const int kHE = tb.he, kHN = tb.hn, kRowMax = tb.rowmax;
  int* tabE = sm;
  int* tabN = sm + kHE;
  int* list = tabN + kHN;
  __shared__ int nlist;
  if (FILL && *ovf) return;
  for (int i = blockIdx.x; i < cD.J; i += gridDim.x) {
    const int a = cD.ni_off[i], b = cD.ni_off[i + 1];
    // a node none of whose incident elements has pairs here or is a partner
    // (a rank's local pattern: most nodes) has an empty row: skip the tables
    bool any = false;
    for (int k = a; k < b && !any; ++k) {
      const int T = cD.ni_el[k], lo = cD.ipos[T];
      any = (lo >= plo && lo < phi) || (pmark && pmark[T]);
    }
    if (!any) {
      if (MODE != 1 && threadIdx.x == 0) rlen[i] = 0;
      if (MODE == 2 && threadIdx.x == 0) roff[i] = 0;
      continue;
    }
    for (int s = threadIdx.x; s < kHE; s += blockDim.x) tabE[s] = -1;
    for (int s = threadIdx.x; s < kHN; s += blockDim.x) tabN[s] = -1;
    if (threadIdx.x == 0) nlist = 0;
    __syncthreads();
    for (int k = a; k < b; ++k) {
      const int T = cD.ni_el[k];
      const int lo = cD.ipos[T];
      if (pmark && pmark[T] && threadIdx.x == 0) hset_insert(tabE, kHE, T, ovf);
      if (lo < plo || lo >= phi) continue;
      const long long p0 = pair_off[lo], p1 = pair_off[lo + 1];
      for (long long p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const int Tp = partner[p];
        if (cD.region[Tp] == 0) hset_insert(tabE, kHE, Tp, ovf);
      }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < kHE; s += blockDim.x) {
      const int Tp = tabE[s];
      if (Tp < 0) continue;
      const int4 w = cD.verts[Tp];
      const int vv[4] = {w.x, w.y, w.z, w.w};
      for (int q = 0; q < 4; ++q)
        if (hset_insert(tabN, kHN, vv[q], ovf)) {
          const int pos = atomicAdd(&nlist, 1);
          if (pos < kRowMax) list[pos] = vv[q];
          else *ovf = 1;
        }
    }
    __syncthreads();
    const int n = nlist < kRowMax ? nlist : kRowMax;
    if (MODE == 0) {
      if (threadIdx.x == 0) rlen[i] = n;
    } else if (MODE == 1) {
      block_sort(list, n);
      const long long o = roff[i];
      for (int s = threadIdx.x; s < n; s += blockDim.x) rcols[o + s] = list[s];
    } else {
      __shared__ long long srow;
      if (threadIdx.x == 0) {
        srow = (long long)atomicAdd(cursor, (unsigned long long)n);
        roff[i] = srow;
        rlen[i] = n;
      }
      block_sort(list, n);
      __syncthreads();
      const long long o = srow;
      if (o + n <= cap)
        for (int s = threadIdx.x; s < n; s += blockDim.x) rcols[o + s] = list[s];
      else if (threadIdx.x == 0)
        atomicCAS(ovf, 0, kCapRetry);
    }
    __syncthreads();
  }
}

// single-pass rows: the total (the cursor) becomes roff[J]
__global__ void k_rows_total(const unsigned long long* cursor, long long* total) {
  *total = (long long)*cursor;
}

__global__ void k_col_count(const long long* total, const int* cols, int* cnt, const int* ovf) {
  if (*ovf) return;
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < *total) atomicAdd(cnt + cols[k], 1);
}

// warp per row: lanes scatter the row's entries into the transposed rows
__global__ void k_transpose_fill(int J, const long long* roff, const int* rlen, const int* rcols,
                                 const long long* toff, int* cursor, int* tcols, const int* ovf) {
  const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= J || *ovf) return;
  const long long rend = rlen ? roff[i] + rlen[i] : roff[i + 1];  // (rows in arrival order)
  for (long long k = roff[i] + (threadIdx.x & 31); k < rend; k += 32) {
    const int j = rcols[k];
    tcols[toff[j] + atomicAdd(cursor + j, 1)] = i;
  }
}

__global__ void __launch_bounds__(256) k_sort_rows(int J, const long long* off, int* cols,
                                                   int* ovf, int kRowMax) {
  extern __shared__ int sm[];
  if (*ovf) return;
  for (int i = blockIdx.x; i < J; i += gridDim.x) {
    const long long a = off[i];
    const int n = (int)(off[i + 1] - a);
    if (n <= 1) continue;
    if (n > kRowMax) {
      if (threadIdx.x == 0) *ovf = 1;
      continue;
    }
    for (int s = threadIdx.x; s < n; s += blockDim.x) sm[s] = cols[a + s];
    __syncthreads();
    block_sort(sm, n);
    for (int s = threadIdx.x; s < n; s += blockDim.x) cols[a + s] = sm[s];
    __syncthreads();
  }
}

__device__ __forceinline__ int lower_bound_int(const int* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// S(i) = R(i) ∪ R^T(i), both sorted.  CTA per row: flag the R^T entries absent
// from R, exclusive-scan the flags in shared memory; then every entry knows its
// merged position from one binary search (R[a] -> a + #new R^T below it,
// new R^T[b] -> #R below it + #new R^T before b).
constexpr int kUnionThreads = 128;
template <bool FILL>
__global__ void __launch_bounds__(kUnionThreads) k_union(int J, const long long* roff,
                                                         const int* rlen,
                                                         const int* rcols, const long long* toff,
                                                         const int* tcols, int* slen,
                                                         const long long* soff, int* scols,
                                                         int* maxlen, const int* ovf,
                                                         int kRowMax) {
  extern __shared__ int pre[];  // kRowMax + 1
  __shared__ int wtot[kUnionThreads / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (*ovf) return;
  for (int i = blockIdx.x; i < J; i += gridDim.x) {
    const long long a0 = roff[i], b0 = toff[i];
    const int na = rlen ? rlen[i] : (int)(roff[i + 1] - a0), nb = (int)(toff[i + 1] - b0);
    if (nb > kRowMax) continue;  // flagged by k_sort_rows
    const int* R = rcols + a0;
    const int* RT = tcols + b0;
    const int c = (nb + kUnionThreads - 1) / kUnionThreads;
    const int lo = min(t * c, nb), hi = min(lo + c, nb);
    int cnt = 0;
    for (int b = lo; b < hi; ++b) {
      const int x = RT[b];
      const int l = lower_bound_int(R, na, x);
      const int f = (l < na && R[l] == x) ? 0 : 1;
      pre[b] = f;
      cnt += f;
    }
    int inc = cnt;
    for (int sh = 1; sh < 32; sh <<= 1) {
      const int y = __shfl_up_sync(FULLMASK, inc, sh);
      if (lane >= sh) inc += y;
    }
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    int run = inc - cnt, total = 0;
    for (int w = 0; w < kUnionThreads / 32; ++w) {
      if (w < wid) run += wtot[w];
      total += wtot[w];
    }
    for (int b = lo; b < hi; ++b) {
      const int f = pre[b];
      pre[b] = run;
      run += f;
    }
    if (t == 0) pre[nb] = total;
    __syncthreads();
    if (!FILL) {
      if (t == 0) {
        slen[i] = na + total;
        atomicMax(maxlen, na + total);
      }
    } else {
      const long long o = soff[i];
      for (int a = t; a < na; a += kUnionThreads) {
        const int x = R[a];
        scols[o + a + pre[lower_bound_int(RT, nb, x)]] = x;
      }
      for (int b = t; b < nb; b += kUnionThreads)
        if (pre[b + 1] != pre[b]) {
          const int x = RT[b];
          scols[o + lower_bound_int(R, na, x) + pre[b]] = x;
        }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ long long find_slot(const long long* soff, const int* scols, int i,
                                               int j) {
  long long lo = soff[i], hi = soff[i + 1] - 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (scols[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return (lo <= hi && scols[lo] == j) ? lo : -1;
}

// warp per row
__global__ void k_mirror(int J, const long long* soff, const int* scols, long long* mirror,
                         int* ovf) {
  const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= J || *ovf) return;
  for (long long k = soff[i] + (threadIdx.x & 31); k < soff[i + 1]; k += 32) {
    const long long m = find_slot(soff, scols, scols[k], i);
    if (m < 0) *ovf = 2;
    mirror[k] = m;
  }
}

// the 10 (b <= b') slots of each interior element's node pairs, stored at
// row min(M_b, M_b')
__global__ void k_edge_slots(const long long* soff, const int* scols, long long* eslot,
                             int* ovf, int plo, int phi, const unsigned char* pmark) {
  const int ii = blockIdx.x * blockDim.x + threadIdx.x;
  if (ii >= cD.KI || *ovf) return;
  if ((ii < plo || ii >= phi) && !(pmark && pmark[cD.interior[ii]])) {
    // neither an outer element of this pattern nor a partner: never read
    for (int k = 0; k < 10; ++k) eslot[10 * (long long)ii + k] = -1;
    return;
  }
  const int4 w = cD.verts[cD.interior[ii]];
  const int v[4] = {w.x, w.y, w.z, w.w};
  int k = 0;
  for (int b = 0; b < 4; ++b)
    for (int c = b; c < 4; ++c, ++k) {
      const int lo = min(v[b], v[c]), hi = max(v[b], v[c]);
      const long long s = find_slot(soff, scols, lo, hi);
      if (s < 0) *ovf = 3;
      eslot[10 * (long long)ii + k] = s;
    }
}

// output pattern: rows = unknown nodes (dof order), columns = unknown nodes;
// warp per row, ballot compaction keeps the column order
template <bool FILL>
__global__ void k_outpat(const long long* soff, const int* scols, int* olen,
                         const long long* ooff, int* ocols, long long* omap, const int* dof_node,
                         const int* ovf) {
  const int d = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= cD.unknowns || *ovf) return;
  const int i = dof_node[d];
  int n = 0;
  const long long o = FILL ? ooff[d] : 0;
  for (long long base = soff[i]; base < soff[i + 1]; base += 32) {
    const long long k = base + lane;
    const int dj = k < soff[i + 1] ? cD.dof[scols[k]] : -1;
    const unsigned m = __ballot_sync(FULLMASK, dj >= 0);
    if (FILL && dj >= 0) {
      const long long pos = o + n + __popc(m & ((1u << lane) - 1));
      ocols[pos] = dj;
      omap[pos] = k;
    }
    n += __popc(m);
  }
  if (!FILL && lane == 0) olen[d] = n;
}

// ---------------------------------------------------------------------------
// K3/K4: integration + scatter

// Two-word fixed point: x = v*scale (exact: scale is a power of two, |x| < 2^62)
// is split as x = hi + lo * 2^-10 + e with hi = 2^32 rint(x 2^-32) (a multiple
// of 2^32), lo = rint((x - hi) 2^10) (|lo| <= 2^41) and |e| <= 2^-11: an
// accumulated entry resolves 2^-72 of its row bound, and integer adds make the
// sum order-free.  (A single word, rint(x), measured 3.8e-13 of a row's largest
// entry at C4 -- profiles/r2_fixed_point_precision.txt: contributions far below
// one unit vanish systematically; the second word divides that by 2^10.)
//
// Both roundings use the 1.5 * 2^52 magic constant on the FP64 pipe: the
// double <-> int64 conversion instructions (F2I.S64.F64 / I2F.F64.S64) issue on
// the XU pipe at about one lane per clock per SM on sm_100 and held the combine
// at 90% of that pipe (profiles/r2e_combine_ncu.txt) when every contribution
// took three of them.
#ifndef NLFEM_DIAG
#define NLFEM_DIAG 0  // timing diagnostics of the combine (bit 1: no REDs; 2: no item
                      // records; 4: no partner-element gathers) -- wrong results
#endif
constexpr double kFixMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kFixLoScale = 0x1p10, kFixLoInv = 0x1p-10;
__device__ __forceinline__ void red_fixed(unsigned long long* V, long long slot, double v,
                                          double scale) {
  if (NLFEM_DIAG & 1) {
    if (v == 1.2345e300) V[slot & 1] = 1;  // keeps the value live
    return;
  }
  const double x = v * scale;
  const double m1 = fma(x, 0x1p-32, kFixMagic);  // low mantissa word = rint(x 2^-32)
  const int h1 = __double2loint(m1);
  const double r = fma(m1 - kFixMagic, -0x1p32, x);  // exact, |r| <= 2^31
  const double m3 = fma(r, kFixLoScale, kFixMagic);
  const long long lo = __double_as_longlong(m3) - __double_as_longlong(kFixMagic);
  if (h1 != 0) atomicAdd(V + 2 * slot, (unsigned long long)((long long)h1 << 32));
  if (lo != 0) atomicAdd(V + 2 * slot + 1, (unsigned long long)lo);
}

__device__ __forceinline__ double fixed_value(const unsigned long long* V, long long slot,
                                              double iscale) {
  const long long hi = (long long)V[2 * slot], lo = (long long)V[2 * slot + 1];
  return ((double)hi + (double)lo * kFixLoInv) * iscale;
}

// error-free transformation for compensated sums (Knuth TwoSum)
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// butterfly sum over the warp (fixed tree -> deterministic)
__device__ __forceinline__ double wsum(double v) {
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULLMASK, v, s);
  return v;
}

// S2 index of (b, c), b <= c
__device__ __forceinline__ int s2i(int b, int c) { return b * 4 - (b * (b - 1)) / 2 + (c - b); }

__device__ __forceinline__ int interior_pos(int T) { return cD.ipos[T]; }

// Monte Carlo (cap) items of a pair: whole-element caps and straddlers
__device__ __forceinline__ int pair_cap_items(unsigned code) {
  int n = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned c = (code >> (5 * q)) & 31;
    n += (c == kOutCap || (c & kStraddle)) ? 1 : 0;
  }
  return n;
}

// case of a cap item: 0 = whole element T' (outside cap), m = 1..3 inside
// vertices of a straddler (k_mc is specialised on it)
__device__ __forceinline__ int cap_case(unsigned c) {
  return c == kOutCap ? 0 : __popc(c & 15u);
}



// np bounds the chunk's pairs on the host; the actual end (*pend) is read on
// the device, entries past it count zero
__global__ void k_units_count(long long p0, long long np, const long long* pend,
                              const unsigned* info, int* ucount) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  ucount[i] = (p0 + i < *pend) ? pair_cap_items(info[p0 + i]) : 0;
}


// unit descriptors: pair index (chunk-relative) and (q | sub << 2); unit ids
// are also listed per parent kind (interior / constraint) so each Monte Carlo
// launch runs one code path (list order is irrelevant: every unit writes only
// its own slot)
// Monte Carlo units: one per sub-simplex slot of a cap item (the reference's
// straddle_outer pieces, upper bound 3 or 1 before the volume floor).  Items
// are listed by their first unit id in four lists -- (interior, constraint)
// parent x (1, 3) slots -- so each k_mc launch runs one uniform code path.
// cap items (one record slot each, in pair then q order) into eight lists by
// parent kind (interior / constraint) and cap_case.  Reservation: per-lane
// counts packed 8 bits per list into one 64-bit word (a warp adds at most 128
// per field), one warp scan, then a block prefix and one global atomic per
// list and block.
constexpr int kFillThreads = 256;
// Each list entry is the item's whole descriptor -- (record slot u, outer
// element T, inner element T', q | class code << 8) -- so the units kernels
// reach the element records after one dependent load instead of five
// (list -> pair -> outer position -> interior id / partner / class).
__global__ void __launch_bounds__(kFillThreads) k_units_fill(long long p0, long long np,
                                                             const long long* pend,
                                                             const unsigned* info,
                                                             const long long* uoff,
                                                             const int* pair_outer,
                                                             const int* partner, int4* lists,
                                                             long long lstride, int* nlist) {
  constexpr int W = kFillThreads / 32;
  __shared__ unsigned long long wtot[W];
  __shared__ int bbase[8][W];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = i < np && p0 + i < *pend;
  const unsigned code = act ? info[p0 + i] : 0;
  const int kind0 = (act && cD.region[partner[p0 + i]] != 0) ? 4 : 0;
  unsigned long long packed = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned c = (code >> (5 * q)) & 31;
    if (c == kOutCap || (c & kStraddle)) packed += 1ull << (8 * (kind0 + cap_case(c)));
  }
  unsigned long long incl = packed;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long t = __shfl_up_sync(FULLMASK, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) wtot[wl] = incl;
  __syncthreads();
  if (threadIdx.x < 8) {  // list k: warp offsets within the block, one global atomic
    const int k = threadIdx.x;
    int run = 0;
    for (int w = 0; w < W; ++w) {
      bbase[k][w] = run;
      run += (int)((wtot[w] >> (8 * k)) & 0xff);
    }
    const int g = run ? atomicAdd(nlist + k, run) : 0;
    for (int w = 0; w < W; ++w) bbase[k][w] += g;
  }
  __syncthreads();
  if (!act) return;
  unsigned long long excl = incl - packed;  // bumped per item: same-list items are consecutive
  long long u = uoff[i];
  const int T = cD.interior[pair_outer[i]];
  const int Tp = partner[p0 + i];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const unsigned c = (code >> (5 * q)) & 31;
    if (!(c == kOutCap || (c & kStraddle))) continue;
    const int k = kind0 + cap_case(c);
    const int slot = bbase[k][wl] + (int)((excl >> (8 * k)) & 0xff);
    excl += 1ull << (8 * k);
    lists[k * lstride + slot] = make_int4((int)u, T, Tp, (int)(q | (c << 8)));
    ++u;
  }
}

// outer element of every pair of the chunk: warp per outer element
__global__ void k_pair_outer(int ii0, int ii1, const long long* pair_off, long long P0,
                             int* pair_outer) {
  const int ii = ii0 + (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (ii >= ii1) return;
  for (long long p = pair_off[ii] + (threadIdx.x & 31); p < pair_off[ii + 1]; p += 32)
    pair_outer[p - P0] = ii;
}

// Philox4x32-R (R = NLFEM_MC_ROUNDS, include/nlfem_mc_stream.h) on two
// counters in lockstep (independent chains); the same function as
// nlfem_philox4x32_r applied to each counter.
__device__ __forceinline__ void philox2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t j2,
                                        uint32_t A[4], uint32_t B[4]) {
  uint32_t a0 = c0, a1 = c1, a2 = c2, a3 = j2;
  uint32_t b0 = c0, b1 = c1, b2 = c2, b3 = j2 + 1;
#pragma unroll
  for (int r = 0; r < NLFEM_MC_ROUNDS; ++r) {
    const unsigned long long pa0 = (unsigned long long)NLFEM_PHILOX_M0 * a0;
    const unsigned long long pa2 = (unsigned long long)NLFEM_PHILOX_M1 * a2;
    const unsigned long long pb0 = (unsigned long long)NLFEM_PHILOX_M0 * b0;
    const unsigned long long pb2 = (unsigned long long)NLFEM_PHILOX_M1 * b2;
    // round keys from constant memory: LOP3 reads them as c[][] operands
    const uint32_t kk0 = cD.rkey[2 * r], kk1 = cD.rkey[2 * r + 1];
    a0 = (uint32_t)(pa2 >> 32) ^ a1 ^ kk0; a1 = (uint32_t)pa2;
    a2 = (uint32_t)(pa0 >> 32) ^ a3 ^ kk1; a3 = (uint32_t)pa0;
    b0 = (uint32_t)(pb2 >> 32) ^ b1 ^ kk0; b1 = (uint32_t)pb2;
    b2 = (uint32_t)(pb0 >> 32) ^ b3 ^ kk1; b3 = (uint32_t)pb0;
  }
  A[0] = a0; A[1] = a1; A[2] = a2; A[3] = a3;
  B[0] = b0; B[1] = b1; B[2] = b2; B[3] = b3;
}


// a 21-bit field as an exact double with one DADD: the bits 0x43300000:s are 2^52 + s
// (I2F.F64.U32 instead measured equal)
__device__ __forceinline__ double u21_to_double(uint32_t s) {
  return __hiloint2double(0x43300000, (int)s) - 4503599627370496.0;  // 2^52
}

// the sorted fields of the even / odd sample of a Philox output w[0..3]
// (nlfem_mc_fields, include/nlfem_mc_stream.h): 3-input min / max (VIMNMX3)
// and the median from the sum (exact: the fields are < 2^21)
__device__ __forceinline__ void sorted3(uint32_t f0, uint32_t f1, uint32_t f2, uint32_t& s0,
                                        uint32_t& s1, uint32_t& s2) {
  s0 = min(min(f0, f1), f2);
  s2 = max(max(f0, f1), f2);
  s1 = f0 + f1 + f2 - s0 - s2;
}
__device__ __forceinline__ void fields_even(const uint32_t w[4], uint32_t& s0, uint32_t& s1,
                                            uint32_t& s2) {
  sorted3(w[0] >> 11, w[1] >> 11, w[2] >> 11, s0, s1, s2);
}
__device__ __forceinline__ void fields_odd(const uint32_t w[4], uint32_t& s0, uint32_t& s1,
                                           uint32_t& s2) {
  // (w_t << 10) | bits of w3: a funnel shift and a mask each
  sorted3(__funnelshift_l(w[3], w[0], 10) & 0x1fffffu,
          __funnelshift_l(w[3] << 10, w[1], 10) & 0x1fffffu,
          __funnelshift_l(w[3] << 20, w[2], 10) & 0x1fffffu, s0, s1, s2);
}

// Hit test Q(s) < delta^2 (nlfem_mc_q) and, on a hit, the exact moments of
// the sorted fields: n and sum s in u32 (< 2^21 per sample, <= 1024 samples
// per segment), sum s s^T in u64 -- the products of two fields are integers
// < 2^42, accumulated by IMAD.WIDE.U32 (one instruction each, exact).  The
// fields are masked by the hit bit (zero on a miss), not branched on: the warp
// issues no divergent code.  The products run on the FMA pipe: the FP64 pipe
// keeps only the conversions and the quadratic form (ncu at P3f with them as
// DFMAs: FP64-pipe throttle and dispatch stalls 42% of the loop's samples).
__device__ __forceinline__ unsigned long long imad_wide(uint32_t a, uint32_t b,
                                                        unsigned long long c) {
  return (unsigned long long)a * b + c;
}
// a * b + c as one IMAD (FMA pipe) where the compiler would pick a SEL (ALU)
__device__ __forceinline__ uint32_t imad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

#ifndef NLFEM_MC_MOM
#define NLFEM_MC_MOM 6  // 6: fields masked by one SEL on the high word (-4.8% at C3f);
                        // 4: masked by two LOP3 per field; 0: masked by a DMUL with
                        // the hit bit (2% slower at C2); 1-3: integer products
#endif
#ifndef NLFEM_MC_I2F
#define NLFEM_MC_I2F 2  // bit t: field t converted by I2F.F64.U32 instead of the DADD
#endif

struct IntMoments {
  unsigned n = 0;
  uint32_t s[3] = {0, 0, 0};
#if NLFEM_MC_MOM == 0 || NLFEM_MC_MOM >= 4
  double ss[6] = {0, 0, 0, 0, 0, 0};  // 00 01 02 11 12 22
#else
  unsigned long long ss[6] = {0, 0, 0, 0, 0, 0};  // 00 01 02 11 12 22
#endif
  __device__ __forceinline__ void sample(const nlfem_mc_quad& Q, double dd, uint32_t s0,
                                         uint32_t s1, uint32_t s2) {
    // field 1 by I2F.F64.U32 (XU pipe, otherwise idle), the others by the DADD
    const double d0 = (NLFEM_MC_I2F & 1) ? __uint2double_rn(s0) : u21_to_double(s0);
    const double d1 = (NLFEM_MC_I2F & 2) ? __uint2double_rn(s1) : u21_to_double(s1);
    const double d2 = (NLFEM_MC_I2F & 4) ? __uint2double_rn(s2) : u21_to_double(s2);
    const bool hit = nlfem_mc_q(&Q, d0, d1, d2) < dd;
    const uint32_t hb = hit ? 1u : 0u;
    n += hb;
#if NLFEM_MC_MOM == 0
    s[0] = imad_u32(hb, s0, s[0]);
    s[1] = imad_u32(hb, s1, s[1]);
    s[2] = imad_u32(hb, s2, s[2]);
    const double h = __hiloint2double((int)imad_u32(hb, 0x3ff00000u, 0u), 0);
    const double h0 = h * d0, h1 = h * d1, h2 = h * d2;
    ss[0] = fma(h0, d0, ss[0]);
    ss[1] = fma(h0, d1, ss[1]);
    ss[2] = fma(h0, d2, ss[2]);
    ss[3] = fma(h1, d1, ss[3]);
    ss[4] = fma(h1, d2, ss[4]);
    ss[5] = fma(h2, d2, ss[5]);
#elif NLFEM_MC_MOM == 6
    // a field < 2^21 as a double has a zero low word, so masking the high word
    // alone zeroes it: one SEL per field, in place, both factors masked
    // (ptxas turns hit-predicated DFMAs into DFMA + 2 FSEL, which is slower)
    s[0] = imad_u32(hb, s0, s[0]);
    s[1] = imad_u32(hb, s1, s[1]);
    s[2] = imad_u32(hb, s2, s[2]);
    const double h0 = __hiloint2double(hit ? __double2hiint(d0) : 0, __double2loint(d0));
    const double h1 = __hiloint2double(hit ? __double2hiint(d1) : 0, __double2loint(d1));
    const double h2 = __hiloint2double(hit ? __double2hiint(d2) : 0, __double2loint(d2));
    ss[0] = fma(h0, h0, ss[0]);
    ss[1] = fma(h0, h1, ss[1]);
    ss[2] = fma(h0, h2, ss[2]);
    ss[3] = fma(h1, h1, ss[3]);
    ss[4] = fma(h1, h2, ss[4]);
    ss[5] = fma(h2, h2, ss[5]);
#elif NLFEM_MC_MOM == 4
    // the fields masked in the integer pipe (two LOP3 per double) instead of
    // multiplied by the hit bit on the FP64 pipe
    s[0] = imad_u32(hb, s0, s[0]);
    s[1] = imad_u32(hb, s1, s[1]);
    s[2] = imad_u32(hb, s2, s[2]);
    const uint32_t m = 0u - hb;
    const double h0 = __hiloint2double(__double2hiint(d0) & (int)m, __double2loint(d0) & (int)m);
    const double h1 = __hiloint2double(__double2hiint(d1) & (int)m, __double2loint(d1) & (int)m);
    const double h2 = __hiloint2double(__double2hiint(d2) & (int)m, __double2loint(d2) & (int)m);
    ss[0] = fma(h0, d0, ss[0]);
    ss[1] = fma(h0, d1, ss[1]);
    ss[2] = fma(h0, d2, ss[2]);
    ss[3] = fma(h1, d1, ss[3]);
    ss[4] = fma(h1, d2, ss[4]);
    ss[5] = fma(h2, d2, ss[5]);
#else
#if NLFEM_MC_MOM == 1
    const uint32_t m0 = hb * s0, m1 = hb * s1, m2 = hb * s2;
#else
    const uint32_t m0 = imad_u32(hb, s0, 0u), m1 = imad_u32(hb, s1, 0u),
                   m2 = imad_u32(hb, s2, 0u);
#endif
#if NLFEM_MC_MOM == 3
    s[0] = imad_u32(hb, s0, s[0]);
    s[1] = imad_u32(hb, s1, s[1]);
    s[2] = imad_u32(hb, s2, s[2]);
#else
    s[0] += m0;
    s[1] += m1;
    s[2] += m2;
#endif
    ss[0] = imad_wide(m0, s0, ss[0]);
    ss[1] = imad_wide(m0, s1, ss[1]);
    ss[2] = imad_wide(m0, s2, ss[2]);
    ss[3] = imad_wide(m1, s1, ss[3]);
    ss[4] = imad_wide(m1, s2, ss[4]);
    ss[5] = imad_wide(m2, s2, ss[5]);
#endif
  }
};

// Moments of the hits about x_q from the integer sums: with r = a + F^T s,
//   sum r = n a + g,  g = F^T sum s,
//   sum r r^T = n a a^T + a g^T + g a^T + F^T (sum s s^T) F   (upper 6),
// added to t1 / t2 (FP64); the integer sums are exact, so this is the sum of
// the hits' r and r r^T up to the rounding of these few products.
__device__ __forceinline__ void fold_moments(const nlfem_mc_quad& Q, const IntMoments& im,
                                             double& nh, double t1[3], double t2[6]) {
  const double n = (double)im.n;
  const double S[3] = {(double)im.s[0], (double)im.s[1], (double)im.s[2]};
  double sd[6];  // exact: the sums are < 2^52
#pragma unroll
  for (int k = 0; k < 6; ++k) sd[k] = (double)im.ss[k];
  const double SS[3][3] = {{sd[0], sd[1], sd[2]}, {sd[1], sd[3], sd[4]}, {sd[2], sd[4], sd[5]}};
  double g[3], H[3][3];  // g = F^T S; H[t][y] = sum_u SS[t][u] F[u][y]
#pragma unroll
  // (explicit fma: the translation unit is compiled with -fmad=false for the
  // geometric predicates; this per-piece fold is arithmetic of ours)
  for (int y = 0; y < 3; ++y) {
    g[y] = fma(S[2], Q.F[2][y], fma(S[1], Q.F[1][y], S[0] * Q.F[0][y]));
#pragma unroll
    for (int t = 0; t < 3; ++t)
      H[t][y] = fma(SS[t][2], Q.F[2][y], fma(SS[t][1], Q.F[1][y], SS[t][0] * Q.F[0][y]));
  }
  nh += n;
  double na[3];
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    na[x] = n * Q.a[x];
    t1[x] += na[x] + g[x];
  }
  int k = 0;
#pragma unroll
  for (int x = 0; x < 3; ++x)
#pragma unroll
    for (int y = x; y < 3; ++y, ++k)
      t2[k] += fma(g[x], Q.a[y], fma(Q.a[x], g[y], na[x] * Q.a[y])) +
               fma(Q.F[2][x], H[2][y], fma(Q.F[1][x], H[1][y], Q.F[0][x] * H[0][y]));
}

constexpr long long kMomStride = 10;   // doubles per MC item record (80 B)

// Monte Carlo: one thread per cap item; each kept sub-simplex (piece) gets M
// samples of the mode-P stream (include/nlfem_mc_stream.h).  Writes one record
// per item, at the item's first unit slot (record of kMomStride doubles): the weighted
// S0, then sum w g(y) for constraint parents, or the Cartesian moments about
// v0(T') sum w r' (3) and sum w r' r'^T (6) for interior parents.
constexpr int kMcThreads = 128;

// value, gradient and Hessian at x of a polynomial of total degree <= 2
// (only such g take the moment path in k_mc<true, true>)
__device__ __forceinline__ void poly2_taylor(const Poly& P, Vd x, double& g0, double gr[3],
                                             double H[6]) {
  g0 = poly_eval(P, x);
  gr[0] = gr[1] = gr[2] = 0;
  for (int k = 0; k < 6; ++k) H[k] = 0;
  const double xv[3] = {x.x, x.y, x.z};
  for (int t = 0; t < P.n; ++t) {
    const int e0 = P.e[t][0], e1 = P.e[t][1], e2 = P.e[t][2];
    const int e[3] = {e0, e1, e2};
    const double c = P.c[t];
    // d/dx_a of c x^e: c e_a x^(e - 1_a) (degree <= 2 -> at most one other factor)
    for (int a = 0; a < 3; ++a) {
      if (!e[a]) continue;
      double v = c * e[a];
      for (int b = 0; b < 3; ++b) {
        const int eb = e[b] - (b == a);
        for (int i = 0; i < eb; ++i) v *= xv[b];
      }
      gr[a] += v;
    }
    // Hessian (constant for degree 2): H_aa = 2c (e_a == 2), H_ab = c (e_a = e_b = 1)
    if (e0 + e1 + e2 == 2) {
      int k = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b, ++k)
          H[k] += (a == b) ? (e[a] == 2 ? 2.0 * c : 0.0) : (e[a] == 1 && e[b] == 1 ? c : 0.0);
    }
  }
}

#ifndef NLFEM_MC_MINBLOCKS
#define NLFEM_MC_MINBLOCKS 4
#endif
#ifndef NLFEM_MC_UNROLL
#define NLFEM_MC_UNROLL 1
#endif
constexpr int kMcUnroll = NLFEM_MC_UNROLL;  // Philox blocks in flight per thread

// |det(b - a, c - a, d - a)|: six times tet_volume(a, b, c, d) before its
// division (reference ball_approx.cpp:144-146 divides by 6 after fabs)
__device__ __forceinline__ double tet_det6(Vd a, Vd b, Vd c, Vd d) {
  return fabs(vdot(vcross(vsub(b, a), vsub(c, a)), vsub(d, a)));
}

// A prism A0 A1 A2 | B0 B1 B2 and the volumes of its split
// (A0A1A2B0, A1A2B0B1, A2B0B1B2) (reference ball_approx.cpp:150-155)
struct Prism {
  Vd A0, A1, A2, B0, B1, B2;
  double v[3];
};

__device__ __forceinline__ void prism_volumes(Prism& P) {
  P.v[0] = tet_det6(P.A0, P.A1, P.A2, P.B0) / 6.0;
  P.v[1] = tet_det6(P.A1, P.A2, P.B0, P.B1) / 6.0;
  P.v[2] = tet_det6(P.A2, P.B0, P.B1, P.B2) / 6.0;
}

// split_warped_prism (reference ball_approx.cpp:160-175): the orientation
// whose three volumes sum larger (vb > va swaps A1/A2 and B1/B2).  Decided
// from the undivided determinants when they differ by more than 1e-12
// (far above the few-ulp difference the /6 and the sums can make);
// otherwise from the reference's exact expressions.  The chosen
// orientation's volumes are the split's piece volumes, bit for bit.
__device__ __forceinline__ void warped_prism(Prism& P) {
  const double a0 = tet_det6(P.A0, P.A1, P.A2, P.B0), a1 = tet_det6(P.A1, P.A2, P.B0, P.B1),
               a2 = tet_det6(P.A2, P.B0, P.B1, P.B2);
  const double b0 = tet_det6(P.A0, P.A2, P.A1, P.B0), b1 = tet_det6(P.A2, P.A1, P.B0, P.B2),
               b2 = tet_det6(P.A1, P.B0, P.B2, P.B1);
  const double sa = a0 + a1 + a2, sb = b0 + b1 + b2;
  bool swap;
  if (sb > sa * (1.0 + 1e-12)) swap = true;
  else if (sb < sa * (1.0 - 1e-12)) swap = false;
  else swap = (b0 / 6.0 + b1 / 6.0) + b2 / 6.0 > (a0 / 6.0 + a1 / 6.0) + a2 / 6.0;
  if (swap) {
    const Vd t = P.A1;
    P.A1 = P.A2;
    P.A2 = t;
    const Vd u = P.B1;
    P.B1 = P.B2;
    P.B2 = u;
    P.v[0] = b0 / 6.0;
    P.v[1] = b1 / 6.0;
    P.v[2] = b2 / 6.0;
  } else {
    P.v[0] = a0 / 6.0;
    P.v[1] = a1 / 6.0;
    P.v[2] = a2 / 6.0;
  }
}

// vertex `slot` of element t from its 128-byte element record
__device__ __forceinline__ Vd elem_vertex(int t, int slot) {
  const double* e = reinterpret_cast<const double*>(cD.erec + 4 * (long long)t);
  return {e[4 + 3 * slot], e[5 + 3 * slot], e[6 + 3 * slot]};
}

// One inner piece (Gauss rule, reference AsmSink::sub, assembly.cpp:332-381) of
// a fullcaps straddler, added to the item's record in the Monte Carlo form:
// S0 += vol and (interior parent) the exact Cartesian moments about v0(T'),
// int r' = vol/4 sum_j p'_j, int r' r'^T = vol/20 (sum_j p'_j p'_j^T + s s^T),
// s = sum_j p'_j (the reference's degree-2 rule is exact for lambda and
// lambda lambda^T, which the combine recovers through the barycentric
// Jacobian); (constraint parent) sum_g vol/4 g at the degree-2 points.
template <bool CONS>
__device__ __forceinline__ void inner_piece(Vd a, Vd b, Vd c, Vd d, double vol, double tau,
                                            Vd v0, double* acc, int& kept) {
  if (!(vol > tau)) return;  // push_piece volume floor (ball_approx.cpp:141)
  ++kept;
  acc[0] += vol;
  if (CONS) {
    const Vd pv[4] = {a, b, c, d};
    double sg = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) sg = fma(vol * 0.25, poly_eval(cD.g, quad_point(pv, g)), sg);
    acc[1] += sg;
  } else {
    const Vd q[4] = {vsub(a, v0), vsub(b, v0), vsub(c, v0), vsub(d, v0)};
    const Vd sp = vadd(vadd(q[0], q[1]), vadd(q[2], q[3]));
    const double v4 = vol * 0.25, v20 = vol / 20.0;
    acc[1] += v4 * sp.x;
    acc[2] += v4 * sp.y;
    acc[3] += v4 * sp.z;
    double m2[6] = {sp.x * sp.x, sp.x * sp.y, sp.x * sp.z, sp.y * sp.y, sp.y * sp.z, sp.z * sp.z};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m2[0] = fma(q[j].x, q[j].x, m2[0]);
      m2[1] = fma(q[j].x, q[j].y, m2[1]);
      m2[2] = fma(q[j].x, q[j].z, m2[2]);
      m2[3] = fma(q[j].y, q[j].y, m2[3]);
      m2[4] = fma(q[j].y, q[j].z, m2[4]);
      m2[5] = fma(q[j].z, q[j].z, m2[5]);
    }
#pragma unroll
    for (int kk = 0; kk < 6; ++kk) acc[4 + kk] += v20 * m2[kk];
  }
}

// CONS: constraint parent (accumulates sum g(y) instead of basis moments).
// G2: g has total degree <= 2, so sum_hits g(x_q + r) follows exactly from the
// hit count, sum r and sum r r^T -- the same branch-free moments as interior
// parents -- instead of one polynomial evaluation per hit.
// CASE: 0 = whole element T' (one outer piece); m = 1, 2, 3 inside vertices of a
// straddler -- straddle_inner + straddle_outer (reference ball_approx.cpp:
// 195-298) with every index static: T''s vertices are loaded in crossing order
// (inside slots ascending, then outside slots ascending), crossing k = (i, o)
// at k = i (4 - m) + o.  Outer pieces: m = 1 prism {q0 q1 q2 | w1 w2 w3},
// m = 2 warped prism {w2 q0 q2 | w3 q1 q3}, m = 3 tet (w3 q0 q1 q2); inner
// pieces: m = 1 tet (w0 q0 q1 q2), m = 2 warped prism {w0 q0 q1 | w1 q2 q3},
// m = 3 prism {w0 w1 w2 | q0 q1 q2}.
// OUTER = false (nocaps): the inner pieces only, no Monte Carlo.
template <bool CONS, bool G2, int CASE, bool OUTER = true>
__global__ void __launch_bounds__(kMcThreads, NLFEM_MC_MINBLOCKS) k_mc(long long p0, long long nitems,
                                                      const int4* list, const int* nlistp,
                                                      double* mom, unsigned long long* mc_stats) {
  constexpr int NOUT = !OUTER ? 0 : ((CASE == 1 || CASE == 2) ? 3 : 1);  // outer pieces
  constexpr int NV = CONS ? 2 : 10;                       // record doubles
  // per-thread item state parked in shared memory while the sample loop runs
  // (it keeps only the quadratic form, the moments and the Philox state in
  // registers): the outer pieces' points and volumes, x_q and x_q - v0(T')
  __shared__ double sP[NOUT == 3 ? 18 : (NOUT == 1 ? 12 : 1)][kMcThreads];
  __shared__ double sV[NOUT == 3 ? 3 : 1][kMcThreads];
  __shared__ double sX[OUTER ? 6 : 1][kMcThreads];
  static_assert(OUTER || CASE != 0, "nocaps has no whole-element caps");
  __shared__ double sAcc[NV][kMcThreads];
  unsigned long long draws = 0, hits = 0, led = 0;
  // warps fetch 32 list entries at a time from a per-list cursor (dynamic
  // balance for items of uneven cost); the list length is read on the device,
  // so there is no host round trip between the list fill and this launch
  const int nlist = nlistp[0];
  int* cursor = const_cast<int*>(nlistp) + 8;
  const int lane = threadIdx.x & 31;
  while (true) {
    int base = 0;
    if (lane == 0) base = atomicAdd(cursor, 32);
    base = __shfl_sync(FULLMASK, base, 0);
    if (base >= nlist) break;
    const int li = base + lane;
    if (li >= nlist) continue;
    const int4 dsc = list[li];  // (record slot, T, T', q | code << 8)
    const long long u = dsc.x;
    const int T = dsc.y, Tp = dsc.z;
    const int q = dsc.w & 255;
    const unsigned c = (unsigned)dsc.w >> 8;
    Vd vT[4];
    load_verts(T, vT);
    const Vd xq = quad_point(vT, q);
    const Vd v0P = elem_vertex(Tp, 0);
    const double tau = cD.tau[Tp];
    double acc[NV];
#pragma unroll
    for (int kk = 0; kk < NV; ++kk) acc[kk] = 0.0;
    Vd pa, pb, pc, pd;  // the single outer piece (NOUT == 1)
    double vol1 = 0;
    if constexpr (CASE == 0) {  // whole element (reference assembly.cpp:754-759): no volume floor
      pa = v0P;
      pb = elem_vertex(Tp, 1);
      pc = elem_vertex(Tp, 2);
      pd = elem_vertex(Tp, 3);
      vol1 = tet_det6(pa, pb, pc, pd) / 6.0;
    } else {
      constexpr int m = CASE, mo = 4 - CASE;
      const unsigned mask = c & 15u, om = ~mask & 15u;
      Vd w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = elem_vertex(Tp, j < m ? nth_bit4(mask, j) : nth_bit4(om, j - m));
      // crossing_points (reference geometry.cpp:39-50)
      Vd X[m * mo];
#pragma unroll
      for (int i = 0; i < m; ++i)
#pragma unroll
        for (int o = 0; o < mo; ++o) {
          const Vd a = w[i], b = w[m + o];
          const double t = edge_crossing(a, b, xq, cD.delta);
          X[i * mo + o] = vadd(a, vscale(t, vsub(b, a)));
        }
      int kin = 0;
      if constexpr (CASE == 1) {
        inner_piece<CONS>(w[0], X[0], X[1], X[2], tet_det6(w[0], X[0], X[1], X[2]) / 6.0, tau,
                          v0P, acc, kin);
        if constexpr (OUTER) {
          Prism P{X[0], X[1], X[2], w[1], w[2], w[3], {0, 0, 0}};
          prism_volumes(P);
          const Vd P6[6] = {P.A0, P.A1, P.A2, P.B0, P.B1, P.B2};
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            sP[3 * k][threadIdx.x] = P6[k].x;
            sP[3 * k + 1][threadIdx.x] = P6[k].y;
            sP[3 * k + 2][threadIdx.x] = P6[k].z;
          }
#pragma unroll
          for (int k = 0; k < 3; ++k) sV[k][threadIdx.x] = P.v[k];
        }
      } else if constexpr (CASE == 2) {
        {
          Prism I{w[0], X[0], X[1], w[1], X[2], X[3], {0, 0, 0}};
          warped_prism(I);
          inner_piece<CONS>(I.A0, I.A1, I.A2, I.B0, I.v[0], tau, v0P, acc, kin);
          inner_piece<CONS>(I.A1, I.A2, I.B0, I.B1, I.v[1], tau, v0P, acc, kin);
          inner_piece<CONS>(I.A2, I.B0, I.B1, I.B2, I.v[2], tau, v0P, acc, kin);
        }
        if constexpr (OUTER) {
          Prism P{w[2], X[0], X[2], w[3], X[1], X[3], {0, 0, 0}};
          warped_prism(P);
          const Vd P6[6] = {P.A0, P.A1, P.A2, P.B0, P.B1, P.B2};
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            sP[3 * k][threadIdx.x] = P6[k].x;
            sP[3 * k + 1][threadIdx.x] = P6[k].y;
            sP[3 * k + 2][threadIdx.x] = P6[k].z;
          }
#pragma unroll
          for (int k = 0; k < 3; ++k) sV[k][threadIdx.x] = P.v[k];
        }
      } else {  // CASE == 3
        {
          Prism I{w[0], w[1], w[2], X[0], X[1], X[2], {0, 0, 0}};
          prism_volumes(I);
          inner_piece<CONS>(I.A0, I.A1, I.A2, I.B0, I.v[0], tau, v0P, acc, kin);
          inner_piece<CONS>(I.A1, I.A2, I.B0, I.B1, I.v[1], tau, v0P, acc, kin);
          inner_piece<CONS>(I.A2, I.B0, I.B1, I.B2, I.v[2], tau, v0P, acc, kin);
        }
        pa = w[3];
        pb = X[0];
        pc = X[1];
        pd = X[2];
        vol1 = tet_det6(pa, pb, pc, pd) / 6.0;
      }
      // ledger: straddle_inner (+ straddle_outer) crossings and volumes, Gauss pieces
      if (OUTER)
        led += 2ull * 38ull * (m * mo) + 24ull * (m == 2 ? 18 : 4);
      else
        led += 38ull * (m * mo) + 24ull * (m == 2 ? 9 : (m == 1 ? 1 : 3));
      led += (unsigned long long)kin * (CONS ? 160 : 360);
    }
#pragma unroll
    for (int kk = 0; kk < NV; ++kk) sAcc[kk][threadIdx.x] = acc[kk];
    if constexpr (OUTER) {
      if constexpr (NOUT == 1) {  // park the single outer piece with the prism layout
        const Vd P4[4] = {pa, pb, pc, pd};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sP[3 * k][threadIdx.x] = P4[k].x;
          sP[3 * k + 1][threadIdx.x] = P4[k].y;
          sP[3 * k + 2][threadIdx.x] = P4[k].z;
        }
        sV[0][threadIdx.x] = vol1;
      }
      sX[0][threadIdx.x] = xq.x;
      sX[1][threadIdx.x] = xq.y;
      sX[2][threadIdx.x] = xq.z;
      sX[3][threadIdx.x] = xq.x - v0P.x;  // c0: moments about v0(T')
      sX[4][threadIdx.x] = xq.y - v0P.y;
      sX[5][threadIdx.x] = xq.z - v0P.z;
    }
    const int M = cD.mc;
    const double dd = cD.dd;
    const double otau = CASE == 0 ? -1.0 : tau;
    int kept = 0;
#pragma unroll 1
    for (int k = 0; k < NOUT; ++k) {
      // piece k = prism points k .. k+3 (the single piece: points 0 .. 3)
      auto piece_quad = [&](nlfem_mc_quad& Qp) {
        const int r = 3 * k;
        double v[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int t = 0; t < 3; ++t) v[i][t] = sP[r + 3 * i + t][threadIdx.x];
        const double x[3] = {sX[0][threadIdx.x], sX[1][threadIdx.x], sX[2][threadIdx.x]};
        nlfem_mc_make_quad(v[0], v[1], v[2], v[3], x, &Qp);
      };
      const double vol = sV[k][threadIdx.x];
      if (!(vol > otau)) continue;  // push_piece volume floor (ball_approx.cpp:141)
      const uint32_t c2 = (uint32_t)q | ((uint32_t)kept << 2);
      ++kept;
      const double w = cD.inv_mc > 0 ? vol * cD.inv_mc : vol / M;  // vol / M
      unsigned nh = 0;
      // the item record gains w x (the hits' S0 and moments about v0(T')) --
      // linear in (n, sum r, sum r r^T), so it is added segment by segment
      auto add_moments = [&](unsigned n_u, const double t1[3], const double t2[6]) {
        const double n = (double)n_u;
        nh += n_u;
        double vals[NV];
        vals[0] = w * n;
        if constexpr (CONS) {
          // sum over hits of g(x_q + r) = n g + grad g . sum r + 1/2 sum H_ab r_a r_b
          double g0, gr[3], H[6];
          poly2_taylor(cD.g, {sX[0][threadIdx.x], sX[1][threadIdx.x], sX[2][threadIdx.x]}, g0,
                       gr, H);
          const double quad = 0.5 * (H[0] * t2[0] + H[3] * t2[3] + H[5] * t2[5]) +
                              H[1] * t2[1] + H[2] * t2[2] + H[4] * t2[4];
          vals[1] = w * (n * g0 + gr[0] * t1[0] + gr[1] * t1[1] + gr[2] * t1[2] + quad);
        } else {
          // shift to moments about v0(T'): r' = r + c0, c0 = x_q - v0
          const double c0x = sX[3][threadIdx.x], c0y = sX[4][threadIdx.x],
                       c0z = sX[5][threadIdx.x];
          const double ncx = n * c0x, ncy = n * c0y, ncz = n * c0z;
          vals[1] = w * (t1[0] + ncx);
          vals[2 % NV] = w * (t1[1] + ncy);
          vals[3 % NV] = w * (t1[2] + ncz);
          vals[4 % NV] = w * fma(c0x, 2.0 * t1[0] + ncx, t2[0]);
          vals[5 % NV] = w * fma(c0y, t1[0] + ncx, fma(c0x, t1[1], t2[1]));
          vals[6 % NV] = w * fma(c0z, t1[0] + ncx, fma(c0x, t1[2], t2[2]));
          vals[7 % NV] = w * fma(c0y, 2.0 * t1[1] + ncy, t2[3]);
          vals[8 % NV] = w * fma(c0z, t1[1] + ncy, fma(c0y, t1[2], t2[4]));
          vals[9 % NV] = w * fma(c0z, 2.0 * t1[2] + ncz, t2[5]);
        }
        // item totals: inner pieces, then the kept outer pieces in piece order
#pragma unroll
        for (int kk = 0; kk < NV; ++kk) sAcc[kk][threadIdx.x] += vals[kk];
      };
      // the integer moments of a segment mapped through F and a, recomputed
      // from the parked points (a compiler barrier first: F and a must not stay
      // live in registers across the sample loop)
      auto fold = [&](const IntMoments& im) {
        asm volatile("" ::: "memory");
        nlfem_mc_quad Qf;
        piece_quad(Qf);
        double n = 0, t1[3] = {0, 0, 0}, t2[6] = {0, 0, 0, 0, 0, 0};
        fold_moments(Qf, im, n, t1, t2);
        add_moments(im.n, t1, t2);
      };
      const int full = M >> 2;
      if constexpr (CONS && !G2) {  // g of degree > 2: evaluated at every hit
        nlfem_mc_quad Qd;
        piece_quad(Qd);
        const Vd xs = {sX[0][threadIdx.x], sX[1][threadIdx.x], sX[2][threadIdx.x]};
        unsigned ngh = 0;
        double ng = 0;
        auto one = [&](uint32_t s0, uint32_t s1, uint32_t s2, double ddv) {
          const double d0 = u21_to_double(s0), d1 = u21_to_double(s1), d2 = u21_to_double(s2);
          if (nlfem_mc_q(&Qd, d0, d1, d2) < ddv) {
            double r[3];
            nlfem_mc_r(&Qd, d0, d1, d2, r);
            ++ngh;
            ng += poly_eval(cD.g, {xs.x + r[0], xs.y + r[1], xs.z + r[2]});
          }
        };
        for (int j = 0; j <= full; ++j) {
          const int rem = j < full ? 4 : (M & 3);
          if (rem == 0) break;
          uint32_t A[4], B[4], s0, s1, s2;
          philox2((uint32_t)T, (uint32_t)Tp, c2, 2u * (uint32_t)j, A, B);
          fields_even(A, s0, s1, s2);
          one(s0, s1, s2, dd);
          fields_odd(A, s0, s1, s2);
          one(s0, s1, s2, rem > 1 ? dd : -1.0);
          fields_even(B, s0, s1, s2);
          one(s0, s1, s2, rem > 2 ? dd : -1.0);
          fields_odd(B, s0, s1, s2);
          one(s0, s1, s2, rem > 3 ? dd : -1.0);
        }
        nh = ngh;
        sAcc[0][threadIdx.x] += w * ngh;
        sAcc[1][threadIdx.x] += w * ng;
      } else if constexpr (OUTER) {
        nlfem_mc_quad Qc;  // only the form's coefficients are read in the loop
        piece_quad(Qc);
        // segments of 256 blocks (1024 samples) keep the integer sums exact
        for (int j0 = 0; j0 < full; j0 += 256) {
          IntMoments im;
          const int j1 = min(full, j0 + 256);
#pragma unroll kMcUnroll
          for (int j = j0; j < j1; ++j) {
            uint32_t A[4], B[4], s0, s1, s2;
            philox2((uint32_t)T, (uint32_t)Tp, c2, 2u * (uint32_t)j, A, B);
            fields_even(A, s0, s1, s2);
            im.sample(Qc, dd, s0, s1, s2);
            fields_odd(A, s0, s1, s2);
            im.sample(Qc, dd, s0, s1, s2);
            fields_even(B, s0, s1, s2);
            im.sample(Qc, dd, s0, s1, s2);
            fields_odd(B, s0, s1, s2);
            im.sample(Qc, dd, s0, s1, s2);
          }
          fold(im);
        }
        if (M & 3) {  // partial last block: samples past M are drawn but never hit
          IntMoments im;
          const int rem = M & 3;
          uint32_t A[4], B[4], s0, s1, s2;
          philox2((uint32_t)T, (uint32_t)Tp, c2, 2u * (uint32_t)full, A, B);
          fields_even(A, s0, s1, s2);
          im.sample(Qc, dd, s0, s1, s2);
          fields_odd(A, s0, s1, s2);
          im.sample(Qc, rem > 1 ? dd : -1.0, s0, s1, s2);
          fields_even(B, s0, s1, s2);
          im.sample(Qc, rem > 2 ? dd : -1.0, s0, s1, s2);
          fold(im);
        }
      }
      draws += (unsigned long long)M;
      hits += nh;
      led += 25ull + 35ull * (unsigned long long)M + (CONS ? 12ull : 62ull) * nh;
    }
    // one record per cap item: S0, then sum g (constraint parents) or sum r'
    // and sum r' r'^T (6) about v0(T') (interior parents), inner pieces included
    double2* rec = reinterpret_cast<double2*>(mom + kMomStride * u);
#pragma unroll
    for (int kk = 0; kk < NV; kk += 2)
      rec[kk / 2] = make_double2(sAcc[kk][threadIdx.x], sAcc[kk + 1][threadIdx.x]);
  }
  // statistics
  for (int sh = 16; sh > 0; sh >>= 1) {
    draws += __shfl_xor_sync(FULLMASK, draws, sh);
    hits += __shfl_xor_sync(FULLMASK, hits, sh);
    led += __shfl_xor_sync(FULLMASK, led, sh);
  }
  if ((threadIdx.x & 31) == 0 && (draws | led)) {
    atomicAdd(mc_stats, draws);
    atomicAdd(mc_stats + 1, hits);
    atomicAdd(mc_stats + 2, led);
  }
}

// approxcaps units: one thread per straddling item; the sphere-point hull's
// fan pieces (approx_pieces, geom.cuh) integrated by the degree-2 rule into the
// item record exactly as k_mc<..., OUTER = false> does for nocaps pieces
// (reference straddle_inner(sphere_points = true) + AsmSink::sub,
// ball_approx.cpp:210-229, assembly.cpp:372-381).
template <bool CONS>
__global__ void __launch_bounds__(kMcThreads) k_approx(long long p0, long long nitems,
                                                       const int4* list, const int* nlistp,
                                                       double* mom, unsigned long long* mc_stats) {
  constexpr int NV = CONS ? 2 : 10;
  unsigned long long led = 0;
  const int nlist = nlistp[0];
  for (int li = blockIdx.x * blockDim.x + threadIdx.x; li < nlist; li += gridDim.x * blockDim.x) {
    const int4 dsc = list[li];  // (record slot, T, T', q | code << 8)
    const long long u = dsc.x;
    const int T = dsc.y, Tp = dsc.z;
    const int q = dsc.w & 255;
    const int mask = (int)(((unsigned)dsc.w >> 8) & 15u);
    Vd vT[4], w[4];
    load_verts(T, vT);
    const Vd xq = quad_point(vT, q);
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = elem_vertex(Tp, j);
    const double tau = cD.tau[Tp];
    double acc[NV];
#pragma unroll
    for (int kk = 0; kk < NV; ++kk) acc[kk] = 0.0;
    int kin = 0;
    if (!approx_pieces(w, mask, xq, cD.delta, tau, [&](Vd a, Vd b, Vd c, Vd d, double vol) {
          inner_piece<CONS>(a, b, c, d, vol, tau, w[0], acc, kin);
        }))
      atomicOr(cD.flags, 1ull);
    const int m = __popc(mask);
    led += 38ull * (m * (4 - m)) + 24ull * kin + (unsigned long long)kin * (CONS ? 160 : 360);
    double2* rec = reinterpret_cast<double2*>(mom + kMomStride * u);
#pragma unroll
    for (int kk = 0; kk < NV; kk += 2) rec[kk / 2] = make_double2(acc[kk], acc[kk + 1]);
  }
  for (int sh = 16; sh > 0; sh >>= 1) led += __shfl_xor_sync(FULLMASK, led, sh);
  if ((threadIdx.x & 31) == 0 && led) atomicAdd(mc_stats + 2, led);
}

// load-vector partials: one slot per (interior element, combine warp, node)
constexpr int kRhsWarps = 8;

// shared-memory map: node id -> slots of (N_a, node) in the four staged rows
struct SlotMap {
  int* key;
  short4* val;  // slot offsets within row a (-1: absent); rows hold < 32768 entries
  int mask;
  // slot of key k, or -1 if the table overflowed while it was built (the
  // combine then flags the run; the host sizes the table up or fails cleanly)
  __device__ __forceinline__ int probe(int k) const {
    unsigned h = hash32((unsigned)k) & mask;
    for (int n = 0; n <= mask; ++n) {
      if (key[h] == k) return (int)h;
      h = (h + 1) & mask;
    }
    return -1;
  }
};

// Combine: CTA per outer element T, thread per element pair.  Whole elements
// are closed form here; straddle items (Gauss units) and caps (Monte Carlo
// units) come precomputed.  A shared-memory map from node id to its slots in the
// four T-node rows of the node pattern locates the T x T' block entries; both
// blocks are added as two-word fixed point with integer atomics.
#ifndef NLFEM_INT_MINBLOCKS
#define NLFEM_INT_MINBLOCKS 2
#endif

// 16 bytes of an item record through the read-only path, or zeros when the
// item is absent: a predicated load, not a branch, so the loads of a pair's
// up to four records are independent of one another and of the code tests and
// can all be in flight together (the combine is bound by load latency)
__device__ __forceinline__ double2 rec_word(const double* rec, int k, unsigned has) {
  double2 r;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "mov.f64 %0, 0d0000000000000000;\n\t"
      "mov.f64 %1, 0d0000000000000000;\n\t"
      "@p ld.global.nc.v2.f64 {%0, %1}, [%3];\n\t}"
      : "=d"(r.x), "=d"(r.y)
      : "r"(has), "l"(rec + 2 * k));
  return r;
}

template <int NTHR>
__global__ void __launch_bounds__(NTHR, (NTHR == 256 ? NLFEM_INT_MINBLOCKS : 2 * NLFEM_INT_MINBLOCKS)) k_integrate(
    int ii0, const long long* __restrict__ pair_off, const int* __restrict__ partner,
    const unsigned* __restrict__ info, const long long* __restrict__ soff,
    const int* __restrict__ scols, const long long* __restrict__ eslot,
    unsigned long long* __restrict__ V, double* __restrict__ rhsT,
    const long long* __restrict__ uoff, const double* __restrict__ mom, long long pbase,
    unsigned long long* __restrict__ stats, int hcap, int rowcap, int nelem, int* spread) {
  static_assert(NTHR / 32 <= kRhsWarps, "one rhsT slot per combine warp");
  extern __shared__ unsigned long long sml[];
  SlotMap mp;
  mp.key = reinterpret_cast<int*>(sml);
  mp.val = reinterpret_cast<short4*>(mp.key + hcap);
  mp.mask = hcap - 1;
  __shared__ long long rbase[4];
  __shared__ double sc[4];
  __shared__ int sNT[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // One outer element per CTA (spread == nullptr, grid = nelem); or -- overlap
  // mode, the combine beside the next chunk's units -- exactly one CTA per SM
  // walking the chunk's elements from a shared cursor.  The block scheduler
  // packs CTAs onto SMs, so the grid holds several candidates per SM and every
  // CTA but the first to arrive on its SM leaves at once (spread[1 + smid]
  // counts arrivals, spread[0] is the element cursor; both zeroed per launch).
  __shared__ int s_el;
  if (spread != nullptr) {
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      s_el = atomicAdd(spread + 1 + smid, 1) == 0 ? atomicAdd(spread, 1) : nelem;
    }
    __syncthreads();
  }
  for (int el = spread ? s_el : (int)blockIdx.x; el < nelem;) {
  const int ii = ii0 + el;
  const int T = cD.interior[ii];
  const int4 wT = cD.verts[T];
  const int NT[4] = {wT.x, wT.y, wT.z, wT.w};

  // slot map of the four T-node rows; zero the row accumulators
  for (int h = threadIdx.x; h < hcap; h += blockDim.x) {
    mp.key[h] = -1;
    mp.val[h] = make_short4(-1, -1, -1, -1);
  }
  if (threadIdx.x < 4) rbase[threadIdx.x] = soff[NT[threadIdx.x]];
  __syncthreads();
  for (int a = 0; a < 4; ++a) {
    const long long r0 = soff[NT[a]], r1 = soff[NT[a] + 1];
    for (long long k = r0 + threadIdx.x; k < r1; k += blockDim.x) {
      const int col = scols[k];
      unsigned h = hash32((unsigned)col) & mp.mask;
      int n = 0;
      for (; n <= mp.mask; ++n) {
        const int prev = atomicCAS(mp.key + h, -1, col);
        if (prev == -1 || prev == col) break;
        h = (h + 1) & mp.mask;
      }
      if (n > mp.mask) {  // the four rows' union outgrew the table
        atomicAdd(stats + 7, 1ull);
        continue;
      }
      reinterpret_cast<short*>(mp.val + h)[a] = (short)(k - r0);
    }
  }
  __syncthreads();

  const double wq = 0.25 * cD.vol[T];  // rule.w[k] * vol (reference assembly.cpp:702)
  const double C = cD.C;
  // per-row constants of T, parked in shared memory (broadcast reads; they
  // would otherwise stay live in registers across the pair loop)
  if (threadIdx.x < 4) {
    sc[threadIdx.x] = cD.scale[NT[threadIdx.x]];
    sNT[threadIdx.x] = NT[threadIdx.x];
  }
  __syncthreads();
  // per outer element: sum over pairs of S0_q (constraint parents weigh 2,
  // reference assembly.cpp:419) and of sum_q c_{q,a} Sg_q
  double s0w[4] = {0, 0, 0, 0}, sgc[4] = {0, 0, 0, 0};
  unsigned long long led = 0;

  const long long p0 = pair_off[ii], p1 = pair_off[ii + 1];
  // software pipeline: the next pair's partner, codes and first record are
  // loaded one iteration ahead, so a pair's dependent gathers start at once
  long long p = p0 + threadIdx.x;
  int TpN = 0;
  unsigned codeN = 0;
  long long uN = 0;
  if (p < p1) {
    TpN = (NLFEM_DIAG & 4) ? T : partner[p];
    codeN = info[p];
    uN = (mom != nullptr) ? uoff[p - pbase] : 0;
  }
  for (; p < p1; p += blockDim.x) {
    const int Tp = TpN;
    const unsigned code = codeN;
    long long u = uN;  // first record of the pair
    {
      const long long pn = p + blockDim.x;
      if (pn < p1) {
        TpN = (NLFEM_DIAG & 4) ? T : partner[pn];
        codeN = info[pn];
        uN = (mom != nullptr) ? uoff[pn - pbase] : 0;
      }
    }
    // partner fields through the read-only path (ld.global.nc): the compiler may
    // then move these loads across the fixed-point REDs (no aliasing with V)
    const bool constr = __ldg(cD.region + Tp) != 0;
    const double volP = __ldg(cD.vol + Tp);

    if (constr) {
      // constraint parent: measure and g integral per point (reference
      // assembly.cpp:350-359, 416-427); no matrix block
      const double gb = __ldg(cD.gbar + Tp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned c = (code >> (5 * q)) & 31;
        if (c == 0) continue;
        double S0 = 0, Sg = 0;
        if (c == kWhole) {
          led += 133;
          S0 = volP;
          Sg = gb;
        } else if (mom != nullptr) {
          const double2 r0 =
              *reinterpret_cast<const double2*>(mom + kMomStride * ((NLFEM_DIAG & 2) ? 0 : u));
          ++u;
          S0 = r0.x;
          Sg = r0.y;
        }
        s0w[q] += 2.0 * S0;
#pragma unroll
        for (int a = 0; a < 4; ++a) sgc[a] += Sg * qbary(q, a);
      }
      continue;
    }

    // interior parent.  The basis moments of an item are an affine image of
    // its Cartesian moments about v0(T') (lambda(y) = e_0 + J (y - v0)), and
    // the pair's blocks are linear in them: X[a][b] = sum_q c_{q,a} S1_q[b],
    // S2 = sum_q S2_q.  So the records are summed over the points first --
    // n0_q and m1_q per point (the point weights c_{q,a} differ), the second
    // moments altogether -- and mapped through J once per pair.
    double n0q[4] = {0, 0, 0, 0}, m1q[4][3], Ms[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) m1q[q][0] = m1q[q][1] = m1q[q][2] = 0;
    double nw = 0;         // whole-element points (a double: no conversion later)
    unsigned wmask = 0;    // ... and which
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned c = (code >> (5 * q)) & 31;
      const bool whole = c == kWhole;
      // straddling / cap item: its record (k_mc: inner pieces, + outer pieces
      // by Monte Carlo for fullcaps); absent items read as zeros
      const unsigned has = (c != 0 && !whole && mom != nullptr) ? 1u : 0u;
      const double* rec = mom + kMomStride * ((NLFEM_DIAG & 2) ? 0 : u);
      u += has;
      const double2 r0 = rec_word(rec, 0, has), r1 = rec_word(rec, 1, has),
                    r2 = rec_word(rec, 2, has), r3 = rec_word(rec, 3, has),
                    r4 = rec_word(rec, 4, has);
      if (whole) {
        led += 39;
        nw += 1.0;
        wmask |= 1u << q;
      }
      n0q[q] = r0.x;
      m1q[q][0] = r0.y;
      m1q[q][1] = r1.x;
      m1q[q][2] = r1.y;
      Ms[0] += r2.x;
      Ms[1] += r2.y;
      Ms[2] += r3.x;
      Ms[3] += r3.y;
      Ms[4] += r4.x;
      Ms[5] += r4.y;
      s0w[q] += whole ? volP : r0.x;
    }

    const int4 wP = __ldg(cD.verts + Tp);
    const int NP[4] = {wP.x, wP.y, wP.z, wP.w};
    const double2 esc01 = __ldg(reinterpret_cast<const double2*>(cD.escale + Tp));
    const double2 esc23 = __ldg(reinterpret_cast<const double2*>(cD.escale + Tp) + 1);
    const double scP[4] = {esc01.x, esc01.y, esc23.x, esc23.y};
    // the ten T' x T' slots, all loaded here (five 16-byte words): issued
    // together instead of one by one between the REDs
    long long es[10];
    {
      const longlong2* ep =
          reinterpret_cast<const longlong2*>(eslot + 10 * (long long)__ldg(cD.ipos + Tp));
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const longlong2 e2 = __ldg(ep + k);
        es[2 * k] = e2.x;
        es[2 * k + 1] = e2.y;
      }
    }

    // J rows from inv_edges, J0 = -(J1+J2+J3)
    const double* invP = cD.inv + 9 * (long long)Tp;
    double J[4][3];
#pragma unroll
    for (int r = 1; r < 4; ++r)
#pragma unroll
      for (int a = 0; a < 3; ++a) J[r][a] = __ldg(invP + 3 * (r - 1) + a);
#pragma unroll
    for (int a = 0; a < 3; ++a) J[0][a] = -(J[1][a] + J[2][a] + J[3][a]);

    const double n0s = (n0q[0] + n0q[1]) + (n0q[2] + n0q[3]);
    double m1s[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) m1s[k] = (m1q[0][k] + m1q[1][k]) + (m1q[2][k] + m1q[3][k]);
    // whole elements: exact basis moments (reference assembly.cpp:361-369)
    const double s1w = volP / 4, offw = nw * (volP / 20.0);
    const double cw = -C * wq;

    // T x T' cross block -C w X[a][b] at (N_a, M_b): shared-memory rows
    {
      double jms[4];  // J_b . sum_q m1_q
#pragma unroll
      for (int b = 0; b < 4; ++b)
        jms[b] = fma(J[b][2], m1s[2], fma(J[b][1], m1s[1], J[b][0] * m1s[0]));
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int hb = mp.probe(NP[b]);
        if (hb < 0) continue;  // overflowed table (flagged above): the run fails
        const short4 sl = mp.val[hb];
        const short sla[4] = {sl.x, sl.y, sl.z, sl.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          // sum_q c_{q,a} S1_q[b], c_{q,a} = QB + (QA - QB) [q == a]
          const double wa = NLFEM_QB * nw + (((wmask >> a) & 1u) ? (NLFEM_QA - NLFEM_QB) : 0.0);
          const double jma = fma(J[b][2], m1q[a][2], fma(J[b][1], m1q[a][1], J[b][0] * m1q[a][0]));
          double xa = fma(NLFEM_QA - NLFEM_QB, jma, NLFEM_QB * jms[b]);
          if (b == 0) xa += fma(NLFEM_QA - NLFEM_QB, n0q[a], NLFEM_QB * n0s);
          const double x = cw * fma(wa, s1w, xa);
          red_fixed(V, rbase[a] + sla[a], sNT[a] == NP[b] ? 2.0 * x : x, sc[a]);
        }
      }
      // T' x T' block C w sum_q S2_q at (M_b, M_c), row min(M_b, M_c)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        double JM[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double m0 = a == 0 ? Ms[0] : (a == 1 ? Ms[1] : Ms[2]);
          const double m1 = a == 0 ? Ms[1] : (a == 1 ? Ms[3] : Ms[4]);
          const double m2 = a == 0 ? Ms[2] : (a == 1 ? Ms[4] : Ms[5]);
          JM[a] = fma(J[b][2], m2, fma(J[b][1], m1, J[b][0] * m0));
        }
#pragma unroll
        for (int cc = b; cc < 4; ++cc) {
          double s2 = fma(JM[2], J[cc][2], fma(JM[1], J[cc][1], JM[0] * J[cc][0]));
          if (b == 0) s2 += jms[cc];
          if (cc == 0) s2 += jms[b];
          if (b == 0 && cc == 0) s2 += n0s;
          s2 += offw * (b == cc ? 2.0 : 1.0);
          red_fixed(V, es[s2i(b, cc)], -cw * s2, NP[b] <= NP[cc] ? scP[b] : scP[cc]);
        }
      }
    }
  }

  // ---- per outer element, per warp (no CTA barrier: a warp that is done
  // leaves): the warp's share of the D_T block as fixed-point REDs (order-free)
  // and of the load vector into its own rhsT slot, which k_finalize adds up
  // in warp order
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    s0w[q] = wsum(s0w[q]);
    sgc[q] = wsum(sgc[q]);
  }
  for (int sh = 16; sh > 0; sh >>= 1) led += __shfl_xor_sync(FULLMASK, led, sh);
  if (lane == 0 && led) atomicAdd(stats + 4, led);  // counter 5: combine ledger
  if (lane < 10) {
    // lanes 0..9: the ten D_T entries (a <= b)
    const int t = lane;
    const int a = t < 4 ? 0 : (t < 7 ? 1 : (t < 9 ? 2 : 3));
    const int b = a + t - (a == 0 ? 0 : (a == 1 ? 4 : (a == 2 ? 7 : 9)));
    double tot = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) tot += C * wq * s0w[q] * qbary(q, a) * qbary(q, b);
    if (tot != 0.0) {
      const int lo = min(sNT[a], sNT[b]), hi = max(sNT[a], sNT[b]);
      int ra = 0;
      for (int r = 0; r < 4; ++r)
        if (sNT[r] == lo) ra = r;
      const int hh = mp.probe(hi);
      const short* v = reinterpret_cast<const short*>(mp.val + (hh < 0 ? 0 : hh));
      red_fixed(V, rbase[ra] + v[ra], tot, sc[ra]);
    }
  } else if (lane < 14) {
    // lanes 10..13: load vector of node a -- f term (reference
    // assembly.cpp:703-709, warp 0 only) + this warp's constraint terms
    const int a = lane - 10;
    double r = 0;
    if (wid == 0) {
      Vd vT[4];
      load_verts(T, vT);
      for (int q = 0; q < 4; ++q) r += wq * qbary(q, a) * poly_eval(cD.f, quad_point(vT, q));
    }
    const double ca = a == 0 ? sgc[0] : (a == 1 ? sgc[1] : (a == 2 ? sgc[2] : sgc[3]));
    rhsT[((long long)ii * kRhsWarps + wid) * 4 + a] = r + 2.0 * C * wq * ca;
  }
  if (spread == nullptr) break;
  __syncthreads();  // every warp is done with this element's map (and has read s_el)
  if (threadIdx.x == 0) s_el = atomicAdd(spread, 1);
  __syncthreads();
  el = s_el;
  }  // elements of this CTA
}


// ---------------------------------------------------------------------------
// K6: fixed point -> CSR values, constraint folding

__global__ void k_finalize(const long long* soff, const int* scols, const long long* mirror,
                           const unsigned long long* V, const long long* ooff,
                           const long long* omap, double* values, const double* rhsT,
                           double* rhs, const int* dof_node, int d0, int d1) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int d = d0 + warp;
  if (d >= d1) return;
  const int i = dof_node[d];
  const double si = cD.iscale[i];
  // matrix entries of output row d: A_ij = V_ij + V_ji (V_ii carries both halves)
  for (long long o = ooff[d] + lane; o < ooff[d + 1]; o += 32) {
    const long long k = omap[o];
    const int j = scols[k];
    double v = fixed_value(V, k, si);
    if (j != i) v += fixed_value(V, mirror[k], cD.iscale[j]);
    values[o] = v;
  }
  // folding of constrained columns: rhs_i -= A_ij g(x_j) (dense-oracle form,
  // reference tests/support/oracles.cpp:274-292), compensated
  double fs = 0, fe = 0;
  for (long long k = soff[i] + lane; k < soff[i + 1]; k += 32) {
    const int j = scols[k];
    if (cD.dof[j] >= 0) continue;
    double v = fixed_value(V, k, si);
    if (j != i) v += fixed_value(V, mirror[k], cD.iscale[j]);
    const Vd x = {cD.node[3 * (long long)j], cD.node[3 * (long long)j + 1], cD.node[3 * (long long)j + 2]};
    double s, e;
    two_sum(fs, v * poly_eval(cD.g, x), s, e);
    fs = s;
    fe += e;
  }
  for (int sh = 16; sh > 0; sh >>= 1) {
    const double os = __shfl_xor_sync(FULLMASK, fs, sh), oe = __shfl_xor_sync(FULLMASK, fe, sh);
    double s, e;
    two_sum(fs, os, s, e);
    fs = s;
    fe += e + oe;
  }
  if (lane == 0) {
    double rs = 0, re = 0;
    for (int k = cD.ni_off[i]; k < cD.ni_off[i + 1]; ++k) {
      const int T = cD.ni_el[k];
      const int lo = cD.ipos[T];
      const int4 w = cD.verts[T];
      const int a = w.x == i ? 0 : (w.y == i ? 1 : (w.z == i ? 2 : 3));
      for (int w = 0; w < kRhsWarps; ++w) {
        double s, e;
        two_sum(rs, rhsT[((long long)lo * kRhsWarps + w) * 4 + a], s, e);
        rs = s;
        re += e;
      }
    }
    double s, e;
    two_sum(rs, -fs, s, e);
    rhs[d] = s + (e + re - fe);
  }
}

// ---------------------------------------------------------------------------
// Owner-computes multi-GPU: a rank integrates its outer
// elements into its local pattern, then ships every local slot of an unknown
// row to that row's owner as a record (key = row << 32 | col; direct hi / lo
// words and the mirror slot's hi / lo), and the rhsT rows of its outer
// elements to the owners of their unknown nodes.  The owner sorts the records
// it receives (its own included), sums equal keys as integers (exact and
// order-free) and finalizes its row block from the merged rows -- the merged
// row of node i is the global pattern row of i, so the result is bit for bit
// the one-GPU system.

// records per unknown row: the local pattern row length
__global__ void k_halo_count(const long long* soff, const int* dof_node, int* cnt) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= cD.unknowns) return;
  const int i = dof_node[d];
  cnt[d] = (int)(soff[i + 1] - soff[i]);
}

// warp per unknown row: one record per local slot
__global__ void k_halo_fill(const long long* soff, const int* scols, const long long* mirror,
                            const unsigned long long* V, const int* dof_node,
                            const long long* hoff, unsigned long long* keys, long long* vals) {
  const int d = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (d >= cD.unknowns) return;
  const int i = dof_node[d];
  const long long s0 = soff[i], o = hoff[d];
  for (long long k = s0 + (threadIdx.x & 31); k < soff[i + 1]; k += 32) {
    const int j = scols[k];
    const long long r = o + (k - s0);
    keys[r] = ((unsigned long long)(unsigned)i << 32) | (unsigned)j;
    longlong2 dv = make_longlong2((long long)V[2 * k], (long long)V[2 * k + 1]);
    longlong2 mv = make_longlong2(0, 0);
    if (j != i) {
      const long long m = mirror[k];
      mv = make_longlong2((long long)V[2 * m], (long long)V[2 * m + 1]);
    }
    reinterpret_cast<longlong2*>(vals)[2 * r] = dv;
    reinterpret_cast<longlong2*>(vals)[2 * r + 1] = mv;
  }
}

__device__ __forceinline__ int owner_of(int d, const int* bounds, int world) {
  int r = 0;
  while (r + 1 < world && d >= bounds[r + 1]) ++r;
  return r;
}

// per outer element of [plo, phi): the ranks owning one of its unknown nodes
__global__ void k_rhs_mask(int plo, int phi, const int* bounds, int world,
                           unsigned long long* mask) {
  const int ii = plo + blockIdx.x * blockDim.x + threadIdx.x;
  if (ii >= phi) return;
  const int4 w = cD.verts[cD.interior[ii]];
  const int v[4] = {w.x, w.y, w.z, w.w};
  unsigned long long m = 0;
  for (int k = 0; k < 4; ++k) {
    const int d = cD.dof[v[k]];
    if (d >= 0) m |= 1ull << owner_of(d, bounds, world);
  }
  mask[ii - plo] = m;
}

__global__ void k_rhs_flag(int n, const unsigned long long* mask, int r, int* flag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) flag[t] = (int)((mask[t] >> r) & 1ull);
}

__global__ void k_rhs_scatter(int n, int plo, const int* flag, const long long* off,
                              long long base, const double* rhsT, int* idx, double* vals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || !flag[t]) return;
  const long long pos = base + off[t];
  idx[pos] = plo + t;
  const double* src = rhsT + (long long)(plo + t) * (4 * kRhsWarps);
  for (int k = 0; k < 4 * kRhsWarps; ++k) vals[pos * (4 * kRhsWarps) + k] = src[k];
}

__global__ void k_rhs_install(long long m, const int* idx, const double* vals, double* rhsT) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * (4 * kRhsWarps)) return;
  const long long r = t / (4 * kRhsWarps), k = t % (4 * kRhsWarps);
  rhsT[(long long)idx[r] * (4 * kRhsWarps) + k] = vals[t];
}

__global__ void k_iota(long long n, unsigned* a) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) a[t] = (unsigned)t;
}

__global__ void k_key_flag(long long n, const unsigned long long* keys, int* flag) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) flag[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1 : 0;
}

__global__ void k_key_start(long long n, const int* flag, const long long* uid, long long* start) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n && flag[t]) start[uid[t]] = t;
  if (t == 0) start[uid[n]] = n;
}

// thread per distinct key: integer sums of its records (any order: exact)
__global__ void k_key_sum(long long nu, const long long* start, const unsigned long long* keys,
                          const unsigned* perm, const long long* vals,
                          unsigned long long* mV, int* mcols, long long* mmirror, int* mcnt) {
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  unsigned long long w[4] = {0, 0, 0, 0};
  for (long long k = start[u]; k < start[u + 1]; ++k) {
    const longlong2* r = reinterpret_cast<const longlong2*>(vals) + 2 * (long long)perm[k];
    const longlong2 a = r[0], b = r[1];
    w[0] += (unsigned long long)a.x;
    w[1] += (unsigned long long)a.y;
    w[2] += (unsigned long long)b.x;
    w[3] += (unsigned long long)b.y;
  }
  const unsigned long long key = keys[start[u]];
  mV[2 * u] = w[0];
  mV[2 * u + 1] = w[1];
  mV[2 * (nu + u)] = w[2];
  mV[2 * (nu + u) + 1] = w[3];
  mcols[u] = (int)(key & 0xffffffffu);
  mmirror[u] = nu + u;
  atomicAdd(mcnt + (int)(key >> 32), 1);
}

// ---------------------------------------------------------------------------
// FP64 DFMA throughput microbenchmark (roofline denominator)

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

// ---------------------------------------------------------------------------
// host side

// Checked build (-DNLFEM_CHECKED=1; compute-sanitizer is closed on this GPU
// pool): every device buffer gets 4-KiB canaries on both sides, and each run
// ends by verifying every live buffer's canaries -- an out-of-bounds write by
// any kernel fails the run with the buffer's size (a bounded substitute for
// memcheck's write checking).  Zero cost in the default build.
#ifndef NLFEM_CHECKED
#define NLFEM_CHECKED 0
#endif
constexpr size_t kGuardBytes = NLFEM_CHECKED ? 4096 : 0;
constexpr unsigned char kGuardByte = 0xA5;
struct GuardEntry {
  char** p;
  size_t* n;
  size_t esz;
};
std::mutex g_guard_mu;
std::map<const void*, GuardEntry> g_guards;
void guard_register(const void* obj, char** p, size_t* n, size_t esz) {
  std::lock_guard<std::mutex> g(g_guard_mu);
  g_guards[obj] = GuardEntry{p, n, esz};
}
void guard_unregister(const void* obj) {
  std::lock_guard<std::mutex> g(g_guard_mu);
  g_guards.erase(obj);
}
// returns a description of the first buffer whose canaries changed, or ""
std::string guard_check() {
  if (!kGuardBytes) return "";
  std::lock_guard<std::mutex> g(g_guard_mu);
  std::vector<unsigned char> h(2 * kGuardBytes);
  for (const auto& kv : g_guards) {
    const GuardEntry& e = kv.second;
    if (!*e.p) continue;
    const size_t bytes = *e.n * e.esz;
    if (cudaMemcpy(h.data(), *e.p - kGuardBytes, kGuardBytes, cudaMemcpyDeviceToHost) !=
            cudaSuccess ||
        cudaMemcpy(h.data() + kGuardBytes, *e.p + bytes, kGuardBytes, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
      return "canary read failed";
    for (size_t i = 0; i < h.size(); ++i)
      if (h[i] != kGuardByte)
        return "buffer of " + std::to_string(*e.n) + " x " + std::to_string(e.esz) +
               " B: canary byte " + std::to_string(i) + (i < kGuardBytes ? " before" : " after") +
               " the buffer overwritten";
  }
  return "";
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t m) {
    if (m <= n && p) return;
    release();
    const size_t bytes = std::max<size_t>(m, 1) * sizeof(T);
    char* base = nullptr;
    CK(cudaMalloc(&base, bytes + 2 * kGuardBytes));
    if (kGuardBytes) {  // checked build: canaries on both sides
      CK(cudaMemset(base, kGuardByte, kGuardBytes));
      CK(cudaMemset(base + kGuardBytes + bytes, kGuardByte, kGuardBytes));
      guard_register(this, reinterpret_cast<char**>(&p), &n, sizeof(T));
    }
    p = reinterpret_cast<T*>(base + kGuardBytes);
    n = std::max<size_t>(m, 1);
  }
  void upload(const T* h, size_t m, cudaStream_t s) {
    ensure(m);
    if (m) CK(cudaMemcpyAsync(p, h, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void release() {
    if (p) cudaFree(reinterpret_cast<char*>(p) - kGuardBytes);
    p = nullptr;
    n = 0;
  }
  ~DBuf() {
    release();
    if (kGuardBytes) guard_unregister(this);
  }
};

// pinned host staging buffer (grow-only): host<->device copies run from
// page-locked memory at full PCIe/C2C rate and asynchronously
struct HostStage {
  char* p = nullptr;
  size_t cap = 0, off = 0;
  void reset(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      CK(cudaMallocHost(reinterpret_cast<void**>(&p), bytes));
      cap = bytes;
    }
    off = 0;
  }
  char* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    if (off + bytes > cap) throw Fail{NLFEM_GPU_ENOMEM, "host staging buffer overflow"};
    char* r = p + off;
    off += bytes;
    return r;
  }
  template <class T>
  void up(DBuf<T>& d, const T* h, size_t m, cudaStream_t s) {
    d.ensure(m);
    if (!m) return;
    char* b = take(m * sizeof(T));
    std::memcpy(b, h, m * sizeof(T));
    CK(cudaMemcpyAsync(d.p, b, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  ~HostStage() {
    if (p) cudaFreeHost(p);
  }
};

// Process-wide pool of page-locked host blocks for the CSR arrays the library
// returns: the download is a straight DMA into the caller's result (no
// staging copy); nlfem_gpu_free_csr hands the block back for the next call.
struct PinnedPool {
  struct Blk {
    char* p;
    size_t n;
    bool used;
  };
  std::mutex mu;
  std::vector<Blk> blks;
  char* acquire(size_t n) {
    std::lock_guard<std::mutex> g(mu);
    Blk* best = nullptr;
    for (auto& b : blks)
      if (!b.used && b.n >= n && (!best || b.n < best->n)) best = &b;
    if (best) {
      best->used = true;
      return best->p;
    }
    char* p = nullptr;
    CK(cudaMallocHost(reinterpret_cast<void**>(&p), std::max<size_t>(n, 256)));
    blks.push_back({p, std::max<size_t>(n, 256), true});
    return p;
  }
  bool release(const void* p) {
    std::lock_guard<std::mutex> g(mu);
    for (auto& b : blks)
      if (b.p == p) {
        b.used = false;
        return true;
      }
    return false;
  }
};
PinnedPool g_result_pool;

}  // namespace

struct nlfem_gpu_session {
  int device = 0;
  int sms = 148;  // streaming multiprocessors of the device (grid sizing)
  int smem_per_sm = 233472;  // shared memory per SM (overlap-mode residency)
  Dev dev{};
  int K = 0, J = 0, KI = 0, unknowns = 0;
  std::vector<int> h_interior, h_dof_node;
  // mesh buffers
  DBuf<double> node, center, radius, vol, tau, inv, diam;
  DBuf<int4> verts, nbr;
  DBuf<uint8_t> region;
  DBuf<int> interior, ipos, dof, dof_node;
  DBuf<double4> erec;
  DBuf<double> gbar, cert2;
  DBuf<unsigned char> bnd;
  // grid / incidence
  DBuf<int> cell_key, cell_cnt, cell_elems, cursor, ni_cnt, ni_el, ai_cnt;
  DBuf<double4> cell_cen;
  DBuf<unsigned long long> ai_vmax;
  DBuf<long long> cell_start64, ni_off64, scan_tmp, scan_tmp2;
  DBuf<int> cell_start, ni_off;
  DBuf<double> scale, iscale;
  DBuf<double4> escale;
  DBuf<unsigned char> econ;
  // pairs
  DBuf<int> pair_count, partner, err_elem, ovf, cand_count, cpartner, spread;
  DBuf<long long> cand_off;
  DBuf<unsigned> cinfo;
  DBuf<unsigned> info;
  DBuf<long long> pair_off;
  DBuf<unsigned long long> counters;
  // pattern
  DBuf<int> rlen, rcols, tcnt, tcols, slen, scols, olen, ocols;
  DBuf<long long> roff, toff, soff, mirror, eslot, ooff, omap;
  // Monte Carlo units (per chunk)
  // two sets, alternating by chunk: the combine of chunk c (on stream4) reads
  // set c & 1 while the units of chunk c + 1 fill the other
  struct UnitBufs {
    DBuf<int> ucount, pair_outer, nlist;
    DBuf<int4> ulist;  // item descriptors, 8 lists
    DBuf<long long> uoff;
    DBuf<double> mom;
  } ub[2];
  float mc_ms = 0;
  int g_deg = 0;  // total degree of g
  // values
  DBuf<unsigned long long> V;
  DBuf<double> rhsT, values, rhs;
  DBuf<int> rowptr32;
  HostStage stage;
  // results of the last run
  long long npairs = 0, nnz_s = 0, nnz_out = 0;
  // sharded pairs (multi-GPU): this rank's K1 range, its pair count, and whether
  // a gathered pair list of all outer elements is installed for the next run
  int pairs_lo = 0, pairs_hi = 0;
  long long shard_npairs = 0, installed_base = 0;
  bool pairs_installed = false;
  long long survivors = 0;   // K1 survivors of the last build_pairs range (bounds its pairs)
  double delta_over_h = 0;   // delta / cbrt(6 mean element volume)
  DBuf<unsigned> info_own;
  // pattern scope: outer elements [plo, phi) have pairs; plocal: a rank's local
  // pattern (owner-computes multi-GPU), pmark[K] flags the interior partners
  int plo = 0, phi = 0;
  bool plocal = false;
  bool pattern_big = false;  // large pattern tables (delta/h >~ 5), kept once needed
  DBuf<unsigned char> pmark;
  // owner-computes multi-GPU: outgoing slot records (key = row << 32 | col,
  // 4 words: direct hi/lo, mirror hi/lo) grouped by destination rank, outgoing
  // rhsT rows, and the merged rows of this rank's row block
  DBuf<int> hcnt;
  DBuf<long long> hoff;
  DBuf<unsigned long long> hkeys;
  DBuf<long long> hvals;
  DBuf<unsigned long long> rmask;
  DBuf<int> rflag, ridx;
  DBuf<long long> roffs;
  DBuf<double> rvals;
  DBuf<unsigned long long> mkeys;
  DBuf<unsigned> midx, midx2;
  DBuf<int> mflag, mcnt, mcols;
  DBuf<long long> muid, moff, mmirror, mstart;
  DBuf<unsigned long long> mV;
  DBuf<unsigned char> cub_tmp;
  std::atomic<long long> launches{0};
  unsigned long long items = 0, mc_samples = 0, mc_hits = 0, ledger = 0, mc_subs = 0,
                     ledger_units = 0;
  cudaStream_t stream = nullptr;
  // the node pattern is built on a second, higher-priority stream from its own
  // host thread, concurrently with the units / Monte Carlo work on `stream`
  cudaStream_t stream2 = nullptr;
  // Gauss units and the one-piece Monte Carlo lists run on stream3, beside the
  // three-piece Monte Carlo lists on `stream`
  cudaStream_t stream3 = nullptr;
  // the combine runs on stream4, overlapping the next chunk's units
  cudaStream_t stream4 = nullptr;
  std::vector<cudaEvent_t> ev;  // 0..7 phases on stream; 8, 9 pattern on stream2; 10, 11 fork/join;
                                // 12, 13 solve; 14..21 per unit-buffer set: units start / end,
                                // combine ready, combine done (kEvUnits0 + 4 set + k)
  DBuf<double> solx, nodev, study_tmp;  // solve: x, node values, reduction scratch
};

namespace {

// exclusive scan of n counts into out[0..n], out[n] = total; the block sums
// of every recursion level live in persistent session scratch (no allocation)
void scan64_level(nlfem_gpu_session& S, long long* scratch, const void* in, bool in_is_int,
                  long long n, long long* out, cudaStream_t st, size_t scratch_off) {
  const long long nb = (n + kScanBlock - 1) / kScanBlock;
  if (n <= 0) {
    CK(cudaMemsetAsync(out, 0, sizeof(long long), st));
    return;
  }
  long long* sums = scratch + scratch_off;
  long long* sums_scan = sums + nb + 1;
  if (in_is_int)
    k_scan_block<int><<<(unsigned)nb, kScanBlock, 0, st>>>((const int*)in, out, sums, n);
  else
    k_scan_block<long long><<<(unsigned)nb, kScanBlock, 0, st>>>((const long long*)in, out, sums, n);
  ++S.launches;
  if (nb > 1) {
    scan64_level(S, scratch, sums, false, nb, sums_scan, st, scratch_off + 2 * (size_t)(nb + 1));
    k_scan_add<<<(unsigned)nb, kScanBlock, 0, st>>>(out, sums_scan, n);
    ++S.launches;
    CK(cudaMemcpyAsync(out + n, sums_scan + nb, sizeof(long long), cudaMemcpyDeviceToDevice, st));
  } else {
    CK(cudaMemcpyAsync(out + n, sums, sizeof(long long), cudaMemcpyDeviceToDevice, st));
  }
}

void scan64(nlfem_gpu_session& S, const void* in, bool in_is_int, long long n, long long* out,
            cudaStream_t st) {
  if (n > 0 && n <= kScan1Max) {
    if (in_is_int)
      k_scan_one<int><<<1, kScan1Threads, 0, st>>>((const int*)in, out, n);
    else
      k_scan_one<long long><<<1, kScan1Threads, 0, st>>>((const long long*)in, out, n);
    ++S.launches;
    return;
  }
  size_t need = 0;
  for (long long m = n; m > 1; m = (m + kScanBlock - 1) / kScanBlock)
    need += 2 * (size_t)((m + kScanBlock - 1) / kScanBlock + 1);
  DBuf<long long>& tmp = (st == S.stream2) ? S.scan_tmp2 : S.scan_tmp;  // scratch per stream
  if (tmp.n < need + 16) {
    CK(cudaStreamSynchronize(st));  // buffer may be in use by queued work
    tmp.ensure(need + 16);
  }
  scan64_level(S, tmp.p, in, in_is_int, n, out, st, 0);
}

long long read_ll(const long long* d, cudaStream_t st) {
  long long h = 0;
  CK(cudaMemcpyAsync(&h, d, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h;
}

__global__ void k_add_offset(long long* a, long long n, long long off) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] += off;
}

__global__ void k_ll_to_int(long long n, const long long* a, int* b) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (int)a[i];
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

void check_config(const nlfem_gpu_kernel* k, const nlfem_gpu_config* cfg) {
  if (!(k->delta > 0)) throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: delta must be positive"};
  if (cfg->mc_samples <= 0)
    throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: mc_samples must be positive"};
  if (cfg->strategy < NLFEM_STRATEGY_INSIDE || cfg->strategy > NLFEM_STRATEGY_FULLCAPS)
    throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: unknown strategy"};
  if (cfg->sampler != NLFEM_SAMPLER_PHILOX)
    throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: unknown sampler"};
}

void poly_to_dev(const nlfem_gpu_poly* p, Poly& d) {
  if (!p) {
    d.n = 0;
    return;
  }
  if (p->nterms > kMaxTerms) throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: polynomial too long"};
  d.n = p->nterms;
  for (int t = 0; t < p->nterms; ++t) {
    d.c[t] = p->coef[t];
    for (int a = 0; a < 3; ++a) d.e[t][a] = p->exps[3 * t + a];
  }
}

void session_init(nlfem_gpu_session& S, const nlfem_gpu_mesh* m, const nlfem_gpu_dofs* dofs,
                  const nlfem_gpu_kernel* k, const nlfem_gpu_poly* f, const nlfem_gpu_poly* g,
                  const nlfem_gpu_config* cfg) {
  check_config(k, cfg);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Fail{NLFEM_GPU_ENODEVICE, "no CUDA device available (the GPU path has no CPU fallback)"};
  if (cfg->device >= 0) CK(cudaSetDevice(cfg->device));
  CK(cudaGetDevice(&S.device));
  CK(cudaDeviceGetAttribute(&S.sms, cudaDevAttrMultiProcessorCount, S.device));
  CK(cudaDeviceGetAttribute(&S.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, S.device));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, S.device));
  if (major < 10)
    throw Fail{NLFEM_GPU_ENODEVICE, "device is not sm_100 class (built for sm_100a only)"};
  if (!S.stream) {  // a reused workspace keeps its streams, events and buffers
    CK(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&S.stream2, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithFlags(&S.stream3, cudaStreamNonBlocking));
#ifndef NLFEM_COMB_PRIO
#define NLFEM_COMB_PRIO 0  // 1: the combine's stream at high priority
#endif
    if (NLFEM_COMB_PRIO)
      CK(cudaStreamCreateWithPriority(&S.stream4, cudaStreamNonBlocking, hi));
    else
      CK(cudaStreamCreateWithFlags(&S.stream4, cudaStreamNonBlocking));
    for (int i = 0; i < 27; ++i) {  // 24..26: overlap-mode probe windows
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      S.ev.push_back(e);
    }
  }
  S.K = m->elem_count;
  S.J = m->node_count;
  S.unknowns = dofs->unknowns;
  if (dofs->node_count != m->node_count)
    throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: dof map does not match the mesh"};
  cudaStream_t st = S.stream;
  // host-side per-element volume floor tau = 1e-14 * diam^3 (reference core.hpp:85)
  std::vector<double> tau(S.K);
  double rmax = 0, dmax = 0;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  double volsum = 0;
  S.h_interior.clear();
  // std::pow (the reference's expression, kept for bit-identical floors) is
  // memoised per distinct diameter: lattice meshes have a handful of shapes
  struct PowMemo {
    uint64_t key[256];
    double val[256];
  } memo;
  std::memset(memo.key, 0xff, sizeof(memo.key));  // NaN pattern: never a diameter
  for (int t = 0; t < S.K; ++t) {
    {
      const double dm = m->diam[t];
      uint64_t b;
      std::memcpy(&b, &dm, 8);
      const unsigned h = (unsigned)((b * 0x9E3779B97F4A7C15ull) >> 56);
      if (memo.key[h] != b) {
        memo.key[h] = b;
        memo.val[h] = 1e-14 * std::pow(dm, 3);
      }
      tau[t] = memo.val[h];
    }
    rmax = std::max(rmax, m->radius[t]);
    dmax = std::max(dmax, m->diam[t]);
    volsum += m->volume[t];
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], m->center[3 * t + a]);
      hi[a] = std::max(hi[a], m->center[3 * t + a]);
    }
    if (!m->region[t]) S.h_interior.push_back(t);
  }
  S.KI = (int)S.h_interior.size();
  std::vector<int> ipos(S.K, -1);
  for (int i = 0; i < S.KI; ++i) ipos[S.h_interior[i]] = i;
  S.h_dof_node.assign(S.unknowns, 0);
  for (int v = 0; v < S.J; ++v)
    if (dofs->dof_of_node[v] >= 0) S.h_dof_node[dofs->dof_of_node[v]] = v;
  // all inputs through the pinned staging buffer, asynchronously
  const size_t K = (size_t)S.K, Jn = (size_t)S.J;
  S.stage.reset(K * (3 * 8 + 8 + 8 + 8 + 72 + 16 + 16 + 1 + 4 + 8) + Jn * (24 + 4) +
                4 * (size_t)S.KI + 4 * (size_t)S.unknowns + 16 * 256);
  S.stage.up(S.node, m->node_xyz, 3 * Jn, st);
  S.stage.up(S.center, m->center, 3 * K, st);
  S.stage.up(S.radius, m->radius, K, st);
  S.stage.up(S.vol, m->volume, K, st);
  S.stage.up(S.diam, m->diam, K, st);
  S.stage.up(S.inv, m->inv_edges, 9 * K, st);
  S.stage.up(S.verts, reinterpret_cast<const int4*>(m->verts), K, st);
  S.stage.up(S.nbr, reinterpret_cast<const int4*>(m->neighbor), K, st);
  S.stage.up(S.region, m->region, K, st);
  S.stage.up(S.dof, dofs->dof_of_node, Jn, st);
  S.stage.up(S.ipos, ipos.data(), K, st);
  S.stage.up(S.tau, tau.data(), K, st);
  S.stage.up(S.interior, S.h_interior.data(), (size_t)S.KI, st);
  S.stage.up(S.dof_node, S.h_dof_node.data(), (size_t)S.unknowns, st);

  Dev& D = S.dev;
  D.K = S.K;
  D.J = S.J;
  D.KI = S.KI;
  D.unknowns = S.unknowns;
  D.strategy = cfg->strategy;
  D.mc = cfg->mc_samples;
  D.seed = cfg->seed;
  D.inv_mc = (cfg->mc_samples > 0 && (cfg->mc_samples & (cfg->mc_samples - 1)) == 0)
                 ? std::ldexp(1.0, -(int)std::log2((double)cfg->mc_samples))
                 : 0.0;
  for (int r = 0; r < 10; ++r) {
    D.rkey[2 * r] = (uint32_t)(cfg->seed & 0xffffffffu) + (uint32_t)r * NLFEM_PHILOX_W0;
    D.rkey[2 * r + 1] = (uint32_t)(cfg->seed >> 32) + (uint32_t)r * NLFEM_PHILOX_W1;
  }
  D.C = k->C;
  D.delta = k->delta;
  D.slack = 1e-10 * k->delta;                           // eps_geo (core.hpp:83)
  D.inside_cut = k->delta - D.slack - 1e-12 * k->delta;  // assembly.cpp:659
  D.dd = k->delta * k->delta;
  poly_to_dev(f, D.f);
  poly_to_dev(g, D.g);
  S.g_deg = 0;
  for (int t = 0; t < D.g.n; ++t)
    S.g_deg = std::max(S.g_deg, D.g.e[t][0] + D.g.e[t][1] + D.g.e[t][2]);
  // uniform grid: cell edge ~ cube root of 6 mean element volumes (one lattice
  // cube holds 6 Kuhn tets), so a cell holds ~6 centers
  const double hg = std::max(std::cbrt(6.0 * volsum / std::max(S.K, 1)), 1e-300);
  D.hg = hg;
  D.ginv = 1.0 / hg;
  D.gox = lo[0];
  D.goy = lo[1];
  D.goz = lo[2];
  D.gx = std::max(1, (int)std::floor((hi[0] - lo[0]) / hg) + 1);
  D.gy = std::max(1, (int)std::floor((hi[1] - lo[1]) / hg) + 1);
  D.gz = std::max(1, (int)std::floor((hi[2] - lo[2]) / hg) + 1);
  D.rmax = rmax;
  S.delta_over_h = S.K > 0 ? k->delta / std::cbrt(6.0 * volsum / S.K) : 0.0;
  S.erec.ensure(4 * (size_t)S.K);
  S.gbar.ensure(S.K);
  S.cert2.ensure(S.K);
  S.bnd.ensure(S.K);
  D.erec = S.erec.p;
  D.gbar = S.gbar.p;
  D.cert2 = S.cert2.p;
  D.bnd = S.bnd.p;
  S.counters.ensure(9);
  D.flags = S.counters.p + 7;
  D.verts = S.verts.p;
  D.nbr = S.nbr.p;
  D.vol = S.vol.p;
  D.tau = S.tau.p;
  D.diam = S.diam.p;
  D.inv = S.inv.p;
  D.region = S.region.p;
  D.interior = S.interior.p;
  D.ipos = S.ipos.p;
  D.dof = S.dof.p;
  D.node = S.node.p;
  (void)dmax;
  // no synchronisation: the inputs sit in the pinned stage, and everything
  // that reads them is ordered after the copies on the same stream
}

// mesh-derived acceleration structures (inside the timed run: the reference's
// equivalent -- interior list, g_node -- is inside its assemble() too)
void run_prep(nlfem_gpu_session& S) {
  cudaStream_t st = S.stream;
  Dev& D = S.dev;
  const int K = S.K, J = S.J;
  const long long ncell = (long long)D.gx * D.gy * D.gz;
  CK(cudaMemcpyToSymbolAsync(cD, &D, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
  S.cell_key.ensure(K);
  S.cell_cnt.ensure(ncell);
  S.cell_elems.ensure(K);
  S.cursor.ensure(std::max<long long>(ncell, J));
  S.cell_start64.ensure(ncell + 1);
  S.cell_start.ensure(ncell + 1);
  S.ni_cnt.ensure(J);
  S.ni_off64.ensure(J + 1);
  S.ni_off.ensure(J + 1);
  S.ai_cnt.ensure(J);
  S.ai_vmax.ensure(J);
  CK(cudaMemsetAsync(S.cell_cnt.p, 0, ncell * sizeof(int), st));
  CK(cudaMemsetAsync(S.ni_cnt.p, 0, J * sizeof(int), st));
  CK(cudaMemsetAsync(S.ai_cnt.p, 0, J * sizeof(int), st));
  CK(cudaMemsetAsync(S.ai_vmax.p, 0, J * sizeof(unsigned long long), st));
  k_elem_prep<<<nblk(K, 256), 256, 0, st>>>(K, S.node.p, S.verts.p, S.center.p, S.radius.p,
                                            S.erec.p, S.gbar.p, S.cert2.p, S.bnd.p, S.cell_key.p,
                                            S.cell_cnt.p, S.ni_cnt.p, S.ai_cnt.p, S.ai_vmax.p);
  ++S.launches;
  // grid: elements sorted by cell (ids ascending within a cell)
  scan64(S, S.cell_cnt.p, true, ncell, S.cell_start64.p, st);
  CK(cudaMemsetAsync(S.cursor.p, 0, ncell * sizeof(int), st));
  k_fill_by_key<<<nblk(K, 256), 256, 0, st>>>(K, S.cell_key.p, S.cell_start64.p, S.cursor.p,
                                              S.cell_elems.p);
  k_sort_segments<<<nblk(ncell, 256), 256, 0, st>>>((int)ncell, S.cell_start64.p, S.cell_elems.p);
  k_ll_to_int<<<nblk(ncell + 1, 256), 256, 0, st>>>(ncell + 1, S.cell_start64.p, S.cell_start.p);
  S.cell_cen.ensure(K);
  k_cell_cen<<<nblk(K, 256), 256, 0, st>>>(K, S.cell_elems.p, S.erec.p, S.cell_cen.p);
  S.launches += 4;
  // node -> interior elements (ascending)
  scan64(S, S.ni_cnt.p, true, J, S.ni_off64.p, st);
  const long long nin = 4LL * S.KI;  // every interior element has 4 nodes: no read-back
  S.ni_el.ensure(nin);
  CK(cudaMemsetAsync(S.cursor.p, 0, J * sizeof(int), st));
  k_ninc_fill<<<nblk(K, 256), 256, 0, st>>>(K, S.ni_off64.p, S.cursor.p, S.ni_el.p);
  k_sort_segments<<<nblk(J, 256), 256, 0, st>>>(J, S.ni_off64.p, S.ni_el.p);
  k_ll_to_int<<<nblk(J + 1, 256), 256, 0, st>>>(J + 1, S.ni_off64.p, S.ni_off.p);
  S.launches += 3;
  S.scale.ensure(J);
  S.iscale.ensure(J);
  D.cell_start = S.cell_start.p;
  D.cell_elems = S.cell_elems.p;
  D.cell_cen = S.cell_cen.p;
  D.ni_off = S.ni_off.p;
  D.ni_el = S.ni_el.p;
  D.scale = S.scale.p;
  D.iscale = S.iscale.p;
  S.escale.ensure(std::max(K, 1));
  S.econ.ensure(std::max(K, 1));
  D.escale = S.escale.p;
  D.econ = S.econ.p;
  CK(cudaMemcpyToSymbolAsync(cD, &D, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
  // fixed-point bound per row: every contribution to
  // row i is bounded by C |B(delta + 3 rmax)| times the volume of the elements
  // around node i, at most 5 such terms (X, 2X on the diagonal, D_T', 2 D_T)
  const double rr = D.delta + 3 * D.rmax;
  const double cbound = 6.0 * D.C * (4.0 / 3.0 * M_PI * rr * rr * rr);
  k_scales<<<nblk(J, 256), 256, 0, st>>>(J, S.ai_cnt.p, S.ai_vmax.p, cbound, S.scale.p, S.iscale.p);
  if (K > 0) k_elem_scales<<<nblk(K, 256), 256, 0, st>>>(K, S.scale.p, S.escale.p, S.econ.p);
  S.launches += 2;
}

void run_finalize(nlfem_gpu_session& S, int r0, int r1) {
  cudaStream_t st = S.stream;
  S.values.ensure(S.nnz_out);
  S.rhs.ensure(S.unknowns);
  if (r1 > r0) {
    k_finalize<<<nblk((long long)(r1 - r0) * 32, 128), 128, 0, st>>>(
        S.soff.p, S.scols.p, S.mirror.p, S.V.p, S.ooff.p, S.omap.p, S.values.p, S.rhsT.p,
        S.rhs.p, S.dof_node.p, r0, r1);
    ++S.launches;
  }
}

// One pass of K5.  spec = true: the buffers keep the capacities of an earlier
// run and nothing comes back to the host until the end (a single read-back);
// returns false if a total exceeded its capacity (nothing was written past
// it) so the caller reruns with spec = false, which reads each size back and
// allocates exactly.
bool pattern_pass(nlfem_gpu_session& S, cudaStream_t st, int& maxlen, bool spec) {
  const int KI = S.KI, J = S.J, U = S.unknowns;
  const PatTabs tb = S.pattern_big ? kPatBig : kPatSmall;
  const int kRowMax = tb.rowmax;
  const size_t rows_smem = (size_t)(tb.he + tb.hn + tb.rowmax) * sizeof(int);
  const size_t union_smem = (size_t)(kRowMax + 1) * sizeof(int);
  CK(cudaFuncSetAttribute(k_rows<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem));
  CK(cudaFuncSetAttribute(k_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem));
  CK(cudaFuncSetAttribute(k_rows<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem));
  CK(cudaFuncSetAttribute(k_union<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)union_smem));
  CK(cudaFuncSetAttribute(k_union<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)union_smem));
  CK(cudaFuncSetAttribute(k_sort_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(kRowMax * sizeof(int))));
  CK(cudaMemsetAsync(S.ovf.p, 0, sizeof(int), st));
  S.rlen.ensure(J);
  S.roff.ensure(J + 1);
  const unsigned rgrid = (unsigned)std::min<long long>(J, (long long)S.sms * 16);
  const unsigned char* pm = S.plocal ? S.pmark.p : nullptr;
  long long capR;
  const int* rlenp = nullptr;  // non-null: rows in arrival order (roff[i], rlen[i])
  if (spec) {
    // one pass: the rows take their places in the earlier run's buffer from a
    // cursor (no counting pass; the row sets are built once)
    capR = (long long)std::min(S.rcols.n, S.tcols.n);
    unsigned long long* cur = S.counters.p + 6;  // (the longest-row slot, reset below)
    CK(cudaMemsetAsync(cur, 0, sizeof(unsigned long long), st));
    k_rows<2><<<rgrid, 256, rows_smem, st>>>(S.pair_off.p, S.partner.p, S.rlen.p, S.roff.p,
                                             S.rcols.p, S.ovf.p, S.plo, S.phi, pm, tb, cur, capR);
    k_rows_total<<<1, 1, 0, st>>>(cur, S.roff.p + J);
    S.launches += 2;
    rlenp = S.rlen.p;
  } else {
    k_rows<0><<<rgrid, 256, rows_smem, st>>>(S.pair_off.p, S.partner.p, S.rlen.p, nullptr,
                                             nullptr, S.ovf.p, S.plo, S.phi, pm, tb, nullptr, 0);
    ++S.launches;
    scan64(S, S.rlen.p, true, J, S.roff.p, st);
    capR = read_ll(S.roff.p + J, st);
    S.rcols.ensure(capR);
    S.tcols.ensure(capR);
    k_rows<1><<<rgrid, 256, rows_smem, st>>>(S.pair_off.p, S.partner.p, nullptr, S.roff.p,
                                             S.rcols.p, S.ovf.p, S.plo, S.phi, pm, tb, nullptr, 0);
  }
  // transpose
  S.tcnt.ensure(J);
  S.toff.ensure(J + 1);
  CK(cudaMemsetAsync(S.tcnt.p, 0, J * sizeof(int), st));
  k_col_count<<<nblk(std::max<long long>(capR, 1), 256), 256, 0, st>>>(S.roff.p + J, S.rcols.p,
                                                                      S.tcnt.p, S.ovf.p);
  scan64(S, S.tcnt.p, true, J, S.toff.p, st);
  S.cursor.ensure(J);
  CK(cudaMemsetAsync(S.cursor.p, 0, J * sizeof(int), st));
  k_transpose_fill<<<nblk(32LL * J, 256), 256, 0, st>>>(J, S.roff.p, rlenp, S.rcols.p, S.toff.p,
                                                        S.cursor.p, S.tcols.p, S.ovf.p);
  k_sort_rows<<<rgrid, 256, kRowMax * sizeof(int), st>>>(J, S.toff.p, S.tcols.p, S.ovf.p,
                                                          kRowMax);
  S.launches += 5;
  // union
  S.slen.ensure(J);
  S.soff.ensure(J + 1);
  CK(cudaMemsetAsync(S.counters.p + 6, 0, sizeof(unsigned long long), st));
  int* d_maxlen = reinterpret_cast<int*>(S.counters.p + 6);
  k_union<false><<<rgrid, kUnionThreads, union_smem, st>>>(J, S.roff.p, rlenp, S.rcols.p, S.toff.p, S.tcols.p,
                                                  S.slen.p, nullptr, nullptr, d_maxlen, S.ovf.p,
                                                  kRowMax);
  ++S.launches;
  scan64(S, S.slen.p, true, J, S.soff.p, st);
  long long capS;
  if (spec) {
    capS = (long long)std::min(S.scols.n, S.mirror.n);
    k_cap_check<<<1, 32, 0, st>>>(S.soff.p + J, capS, S.ovf.p);
  } else {
    capS = read_ll(S.soff.p + J, st);
    S.scols.ensure(capS);
    S.mirror.ensure(capS);
  }
  k_union<true><<<rgrid, kUnionThreads, union_smem, st>>>(J, S.roff.p, rlenp, S.rcols.p, S.toff.p, S.tcols.p,
                                                 nullptr, S.soff.p, S.scols.p, nullptr, S.ovf.p,
                                                 kRowMax);
  k_mirror<<<nblk(32LL * J, 256), 256, 0, st>>>(J, S.soff.p, S.scols.p, S.mirror.p, S.ovf.p);
  S.eslot.ensure(10 * (size_t)KI);
  k_edge_slots<<<nblk(KI, 128), 128, 0, st>>>(S.soff.p, S.scols.p, S.eslot.p, S.ovf.p, S.plo,
                                              S.phi, pm);
  S.launches += 3;
  // output pattern
  S.olen.ensure(U);
  S.ooff.ensure(U + 1);
  k_outpat<false><<<nblk(32LL * U, 256), 256, 0, st>>>(S.soff.p, S.scols.p, S.olen.p, nullptr,
                                                       nullptr, nullptr, S.dof_node.p, S.ovf.p);
  ++S.launches;
  scan64(S, S.olen.p, true, U, S.ooff.p, st);
  long long capO;
  if (spec) {
    capO = (long long)std::min(S.ocols.n, S.omap.n);
    k_cap_check<<<1, 32, 0, st>>>(S.ooff.p + U, capO, S.ovf.p);
  } else {
    capO = read_ll(S.ooff.p + U, st);
    S.ocols.ensure(capO);
    S.omap.ensure(capO);
  }
  k_outpat<true><<<nblk(32LL * U, 256), 256, 0, st>>>(S.soff.p, S.scols.p, nullptr, S.ooff.p,
                                                      S.ocols.p, S.omap.p, S.dof_node.p, S.ovf.p);
  ++S.launches;
  // one read-back: flags, sizes, longest row
  long long sz[3] = {0, 0, 0};
  int flags[2] = {0, 0};
  CK(cudaMemcpyAsync(&flags[0], S.ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&flags[1], d_maxlen, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&sz[0], S.roff.p + J, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&sz[1], S.soff.p + J, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&sz[2], S.ooff.p + U, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (flags[0] == kCapRetry) return false;
  if (flags[0] == 1 && !S.pattern_big) {  // a row or a node block outgrew the small tables
    S.pattern_big = true;
    return false;
  }
  if (flags[0])
    throw Fail{NLFEM_GPU_BAD_CONFIG,
               "BadConfig: interaction neighbourhood too large for the pattern kernels (code " +
                   std::to_string(flags[0]) + ")"};
  S.nnz_s = sz[1];
  S.nnz_out = sz[2];
  maxlen = flags[1];
  return true;
}

// K5: the node pattern S (sorted rows), its mirror / edge slots and the output
// pattern.  Runs on its own stream; buffers sized by an earlier run are reused
// speculatively (no host round trips); otherwise sizes are read back.
void run_pattern(nlfem_gpu_session& S, cudaStream_t st, int& maxlen) {
  const bool spec = S.rcols.n > 1 && S.tcols.n > 1 && S.scols.n > 1 && S.mirror.n > 1 &&
                    S.ocols.n > 1 && S.omap.n > 1;
  if (spec && pattern_pass(S, st, maxlen, true)) return;
  if (pattern_pass(S, st, maxlen, false)) return;
  pattern_pass(S, st, maxlen, false);  // again with the large tables
}

// K1 over outer elements [lo, hi) (positions in the ascending interior list):
// pair_count[ii], cand_off[ii], pair_off[ii] are indexed absolutely, offsets are
// relative to the range start (pair_off[lo] = 0); partner / info hold the
// range's pairs in outer order.  Resets the counters and the BallExitsMesh flag.
// K1 classification pass, instantiated per strategy (and WIDE)
template <bool WIDE>
void launch_pairs1(int strategy, unsigned grid, cudaStream_t st, int lo, int hi,
                   const long long* cand_off, long long cand_base, int* cpartner, unsigned* cinfo,
                   int* pair_count, unsigned long long* counters, int* err_elem) {
#define NLFEM_K1_CASE(ST)                                                                     \
  case ST:                                                                                    \
    k_pairs<1, WIDE, ST><<<grid, kPairThreads, 0, st>>>(lo, hi, cand_off, cand_base, nullptr, \
                                                        cpartner, cinfo, pair_count, counters, \
                                                        err_elem);                            \
    break;
  switch (strategy) {
    NLFEM_K1_CASE(NLFEM_STRATEGY_INSIDE)
    NLFEM_K1_CASE(NLFEM_STRATEGY_OVERLAP)
    NLFEM_K1_CASE(NLFEM_STRATEGY_BARYCENTER)
    NLFEM_K1_CASE(NLFEM_STRATEGY_NOCAPS)
    NLFEM_K1_CASE(NLFEM_STRATEGY_APPROXCAPS)
    NLFEM_K1_CASE(NLFEM_STRATEGY_FULLCAPS)
    default:
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: unknown strategy"};
  }
#undef NLFEM_K1_CASE
}

// element pairs per units / combine chunk (bounds the unit buffers; two sets
// are alive at a time).  NLFEM_PAIRS_PER_CHUNK overrides (tests use tiny chunks).
long long pairs_per_chunk() {
  static const long long v = [] {
    const char* e = std::getenv("NLFEM_PAIRS_PER_CHUNK");
    return e ? std::max(1LL, std::atoll(e)) : (8LL << 20);
  }();
  return v;
}

// ranges of at most this many outer elements take the one-element-per-CTA K1
// (NLFEM_PAIRS_WIDE_MAX overrides)
int pairs_wide_max() {
  static const int v = [] {
    const char* e = std::getenv("NLFEM_PAIRS_WIDE_MAX");
    return e ? std::atoi(e) : 1024;
  }();
  return v;
}

void build_pairs(nlfem_gpu_session& S, int lo, int hi) {
  cudaStream_t st = S.stream;
  const int KI = S.KI;
  S.pair_count.ensure(KI);
  S.pair_off.ensure(KI + 1);
  S.err_elem.ensure(1);
  S.ovf.ensure(1);
  S.counters.ensure(9);
  const int big = 0x7fffffff;
  CK(cudaMemcpyAsync(S.err_elem.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(S.ovf.p, 0, sizeof(int), st));
  CK(cudaMemsetAsync(S.counters.p, 0, 9 * sizeof(unsigned long long), st));
  // pass 0: survivors per outer element (cheap superset count)
  S.cand_count.ensure(KI + 1);
  S.cand_off.ensure(KI + 1);
  const int n = hi - lo;
  if (n > 0) {
    k_pairs<0><<<nblk((long long)n, kPairWarps), kPairThreads, 0, st>>>(
        lo, hi, nullptr, 0, S.cand_count.p, nullptr, nullptr, nullptr, nullptr, nullptr);
    ++S.launches;
  }
  // survivor offsets of the range, relative to its start (cand_off[lo] = 0)
  scan64(S, S.cand_count.p + lo, true, n, S.cand_off.p + lo, st);
  std::vector<long long> coffr(n + 1, 0);
  CK(cudaMemcpyAsync(coffr.data(), S.cand_off.p + lo, sizeof(long long) * (n + 1),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // absolute-indexed view: coff[ii] for ii in [lo, hi]
  auto coff = [&](int ii) { return coffr[ii - lo]; };
  S.survivors = coff(hi);
  // pass 1 + compaction, in chunks of outer elements bounded by survivors
  const long long kCandBudget = 1LL << 30;  // 8 GiB of (partner, code) slots
  S.pair_off.ensure(KI + 1);
  if (coff(hi) <= kCandBudget) {
    // one chunk: pairs <= survivors bounds the pair arrays, so the pair total
    // need not come back to the host here (it arrives with the pair offsets
    // the integration phase reads anyway)
    const long long nc = coff(hi);
    S.partner.ensure(std::max<long long>(1, nc));
    S.info.ensure(std::max<long long>(1, nc));
    S.cpartner.ensure(nc + 1);
    S.cinfo.ensure(nc + 1);
    if (n > 0) {
      if (n <= pairs_wide_max())
        launch_pairs1<true>(S.dev.strategy, (unsigned)n, st, lo, hi, S.cand_off.p, 0,
                            S.cpartner.p, S.cinfo.p, S.pair_count.p, S.counters.p, S.err_elem.p);
      else
        launch_pairs1<false>(S.dev.strategy, (unsigned)nblk((long long)n, kPairWarps), st, lo, hi,
                             S.cand_off.p, 0, S.cpartner.p, S.cinfo.p, S.pair_count.p,
                             S.counters.p, S.err_elem.p);
      scan64(S, S.pair_count.p + lo, true, n, S.pair_off.p + lo, st);
      k_pairs_compact<<<nblk((long long)n * 32, 256), 256, 0, st>>>(
          lo, hi, S.cand_off.p, 0, S.cpartner.p, S.cinfo.p, S.pair_off.p, S.partner.p, S.info.p);
      S.launches += 2;
    }
  } else {
    long long cap = std::max<long long>(1, (long long)(0.8 * coff(hi)));
    S.partner.ensure(cap);
    S.info.ensure(cap);
    long long total = 0;
    int c0 = lo;
    while (c0 < hi) {
      int c1 = lo + (int)(std::upper_bound(coffr.begin() + (c0 - lo) + 1, coffr.end(),
                                           coff(c0) + kCandBudget) -
                          coffr.begin()) - 1;
      c1 = std::min(std::max(c1, c0 + 1), hi);
      const long long nc = coff(c1) - coff(c0);
      S.cpartner.ensure(nc + 1);
      S.cinfo.ensure(nc + 1);
      launch_pairs1<false>(S.dev.strategy, (unsigned)nblk((long long)(c1 - c0), kPairWarps), st,
                           c0, c1, S.cand_off.p, coff(c0), S.cpartner.p, S.cinfo.p,
                           S.pair_count.p, S.counters.p, S.err_elem.p);
      ++S.launches;
      // pair offsets of this chunk continue the running total
      scan64(S, S.pair_count.p + c0, true, c1 - c0, S.pair_off.p + c0, st);
      const long long nch = read_ll(S.pair_off.p + c1, st);
      if (total) {
        k_add_offset<<<nblk(c1 - c0 + 1, 256), 256, 0, st>>>(S.pair_off.p + c0, c1 - c0 + 1, total);
        ++S.launches;
      }
      if (total + nch > cap) {  // grow, keeping what is compacted
        cap = (long long)((total + nch) * 1.25) + 1;
        DBuf<int> np_;
        DBuf<unsigned> ni_;
        np_.ensure(cap);
        ni_.ensure(cap);
        if (total) {
          CK(cudaMemcpyAsync(np_.p, S.partner.p, total * sizeof(int), cudaMemcpyDeviceToDevice, st));
          CK(cudaMemcpyAsync(ni_.p, S.info.p, total * sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
        }
        CK(cudaStreamSynchronize(st));
        std::swap(S.partner.p, np_.p);
        std::swap(S.partner.n, np_.n);
        std::swap(S.info.p, ni_.p);
        std::swap(S.info.n, ni_.n);
      }
      k_pairs_compact<<<nblk((long long)(c1 - c0) * 32, 256), 256, 0, st>>>(
          c0, c1, S.cand_off.p, coff(c0), S.cpartner.p, S.cinfo.p, S.pair_off.p, S.partner.p,
          S.info.p);
      ++S.launches;
      total += nch;
      c0 = c1;
    }
  }
  if (n == 0) {
    const long long z = 0;
    CK(cudaMemcpyAsync(S.pair_off.p + lo, &z, sizeof(long long), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
}

// The whole device pipeline.  Outer elements [shard_lo, shard_hi) (positions in
// the ascending interior list) are integrated; pairs and the node pattern are
// built for all of them (every rank holds the same pattern, so the fixed-point
// partial sums of several ranks add up slot by slot).
// local = true (owner-computes multi-GPU): pairs are built
// for [shard_lo, shard_hi) only and the node pattern is this rank's local one
// (rows touched by those pairs, plus the partners' own node pairs).
void run_all(nlfem_gpu_session& S, cudaStream_t user, nlfem_gpu_stats* stats, int shard_lo,
             int shard_hi, bool finalize, bool local = false) {
  cudaStream_t st = S.stream;
  Dev& D = S.dev;
  const auto wall0 = std::chrono::steady_clock::now();
  S.launches = 0;
  if (user) {
    // order after work the caller queued on its stream
    CK(cudaEventRecord(S.ev[7], user));
    CK(cudaStreamWaitEvent(st, S.ev[7], 0));
  }
  CK(cudaEventRecord(S.ev[0], st));

  // ---- K1: pairs (count, scan, fill), unless a gathered pair list of all
  // outer elements has been installed (sharded multi-GPU pairs)
  const int KI = S.KI;
  const int big = 0x7fffffff;
  const bool installed = S.pairs_installed;
  shard_lo = std::max(0, std::min(shard_lo, KI));
  shard_hi = std::max(shard_lo, std::min(shard_hi, KI));
  local = local && !installed;
  S.plocal = local;
  S.plo = local ? shard_lo : 0;
  S.phi = local ? shard_hi : KI;
  if (!installed) {
    run_prep(S);
    CK(cudaEventRecord(S.ev[1], st));
    build_pairs(S, S.plo, S.phi);
    if (local) {
      // interior partners of this rank's pairs (their node pairs join the
      // local pattern); the pair total is bounded by the K1 survivors
      S.pmark.ensure(S.K);
      CK(cudaMemsetAsync(S.pmark.p, 0, S.K, st));
      if (S.survivors > 0) {
        k_mark_partners<<<nblk(S.survivors, 256), 256, 0, st>>>(
            S.survivors, S.pair_off.p + S.phi, S.partner.p, S.pmark.p);
        ++S.launches;
      }
    }
  } else {
    // the device parameter block is per device, not per session: rebind this
    // session's (another session may have run since its pairs were built)
    CK(cudaMemcpyToSymbolAsync(cD, &D, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(S.ev[1], st));
    S.pairs_installed = false;  // one run per installation
  }
  // the pair offsets (hence the total) and the BallExitsMesh flag come back in
  // one round trip, after the pattern work has been handed to its stream
  std::vector<long long> poff(KI + 1, 0);
  int err_elem_h = big;
  CK(cudaEventRecord(S.ev[2], st));

  // ---- K5: pattern, on stream2 from its own host thread (overlaps the units)
  CK(cudaStreamWaitEvent(S.stream2, S.ev[2], 0));
  int maxlen = 0;
  std::exception_ptr pattern_error;
  std::thread pattern_thread([&S, &maxlen, &pattern_error]() {
    try {
      CK(cudaSetDevice(S.device));
      CK(cudaEventRecord(S.ev[8], S.stream2));
      run_pattern(S, S.stream2, maxlen);
      CK(cudaEventRecord(S.ev[9], S.stream2));
    } catch (...) {
      pattern_error = std::current_exception();
    }
  });
  struct Joiner {  // joins on every exit path (exceptions included)
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{pattern_thread};
  bool pattern_ready = false;
  auto wait_pattern = [&]() {
    if (pattern_ready) return;
    pattern_thread.join();
    if (pattern_error) std::rethrow_exception(pattern_error);
    CK(cudaStreamWaitEvent(st, S.ev[9], 0));
    pattern_ready = true;
  };

  // ---- K3/K4: integrate + scatter
  CK(cudaEventRecord(S.ev[3], st));
  S.rhsT.ensure(4 * kRhsWarps * (size_t)KI);
  CK(cudaMemsetAsync(S.rhsT.p, 0, 4 * kRhsWarps * (size_t)KI * sizeof(double), st));
  // combine set-up once the pattern is known: accumulators and the slot-map
  // capacity, a power of two > union of the four rows (<= 4 maxlen)
  int hcap = 64, rowcap = 1;
  size_t ismem = 0;
  bool combine_ready = false;
  auto setup_combine = [&]() {
    if (combine_ready) return;
    combine_ready = true;
    wait_pattern();
    S.V.ensure(2 * (size_t)S.nnz_s);
    CK(cudaMemsetAsync(S.V.p, 0, 2 * S.nnz_s * sizeof(unsigned long long), st));
    // the four rows of an outer element share most columns: their union is
    // far below 4 maxlen (a table overflow is detected and fails the run)
    while (hcap <= 4 * std::max(maxlen, 1)) hcap <<= 1;
    const size_t kSlot = sizeof(int) + sizeof(short4);
    while (hcap * kSlot > 220 * 1024 && hcap > 2 * std::max(maxlen, 1)) hcap >>= 1;
    if (maxlen >= 32768 || hcap * kSlot > 220 * 1024 || hcap <= std::max(maxlen, 1))
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: pattern rows too long for the integration kernel"};
    rowcap = std::max(maxlen, 1);
    ismem = (size_t)hcap * kSlot;
    CK(cudaFuncSetAttribute(k_integrate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem));
    CK(cudaFuncSetAttribute(k_integrate<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem));
  };
  // units phase: nocaps -> Gauss records (k_gauss); fullcaps -> one record per
  // cap item (k_mc, inner pieces included); barycenter -> none
  // units phase: one record per straddling / cap item -- inner pieces (nocaps,
  // fullcaps) and outer pieces by Monte Carlo (fullcaps); none for barycenter
  const bool need_mc = D.strategy == NLFEM_STRATEGY_FULLCAPS;
  // straddling pieces only under nocaps / fullcaps; the other strategies emit
  // whole-element items only
  const bool need_units = D.strategy == NLFEM_STRATEGY_NOCAPS ||
                          D.strategy == NLFEM_STRATEGY_APPROXCAPS ||
                          D.strategy == NLFEM_STRATEGY_FULLCAPS;
  float mc_ms = 0;
  // chunks of outer elements sized so the unit buffers stay bounded.  One
  // chunk needs no host round trip when its first pair and a bound on its
  // pairs are known on the host: a full run (pairs <= K1 survivors) or a
  // sharded run on installed pairs (offset and count from the install).
  const long long kPairsPerChunk = need_units ? pairs_per_chunk() : (1LL << 40);
  const bool full_run = !installed && (local || (shard_lo == 0 && shard_hi == KI));
  const bool own_range = installed && shard_lo == S.pairs_lo && shard_hi == S.pairs_hi;
  const bool fast = (full_run && S.survivors <= kPairsPerChunk) ||
                    (own_range && S.shard_npairs <= kPairsPerChunk);
  // Overlap mode (Monte Carlo runs of more than two chunks): the combine of a
  // chunk runs beside the units of the next one.  The units kernels use no
  // memory pipe and the combine little else, but unit launches at four CTAs per
  // SM hold every register; capped at three (shared-memory padding, -1.7% of
  // their rate at C3f) they leave room for one 128-thread combine CTA per SM.
  constexpr int kMcPadBytes = 57 * 1024;
  // B200: -5.4% of the step at C3f, -2.3% at C2, -4.3% at C4.  The results do
  // not depend on the mode (the same per-element sums; integer accumulation).
  // NLFEM_COMB_OVERLAP: unset or 3 = on, 0 = off, 1 = resident combine only,
  // 2 = padding only, -1 = measured per run (six chunks with, six without,
  // timed on the units' stream, the faster mode for the rest).
  const char* ov_s = std::getenv("NLFEM_COMB_OVERLAP");
  const int overlap_env = ov_s ? atoi(ov_s) : 3;
  const long long shard_pairs_bound =
      full_run ? S.survivors : (own_range ? S.shard_npairs : (1LL << 62));
  const bool overlap_able = need_mc && !fast && shard_pairs_bound > 2 * kPairsPerChunk;
  constexpr int kProbe0 = 2, kProbeLen = 6;  // windows [2, 8) with, [8, 14) without
  const bool probing = overlap_able && overlap_env < 0 &&
                       shard_pairs_bound > (kProbe0 + 2 * kProbeLen + 6) * kPairsPerChunk;
  int ov_bits = overlap_env > 0 ? (overlap_env & 3) : 0;  // this chunk's mode
  bool overlap = overlap_able && ov_bits != 0;
  auto fits_pad = [&]() {
    return 3 * (kMcPadBytes + 1024) + (int)ismem + 2048 <= S.smem_per_sm;
  };
  auto fits_nopad = [&]() {  // 37,888 B: the largest static shared memory of a units kernel
    return 3 * (37888 + 1024) + (int)ismem + 2048 <= S.smem_per_sm;
  };
  bool npairs_pending = false;
  if (fast) {
    npairs_pending = full_run;  // read at the end with the BallExitsMesh flag
  } else {
    CK(cudaMemcpyAsync(poff.data(), S.pair_off.p, sizeof(long long) * (KI + 1),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&err_elem_h, S.err_elem.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err_elem_h != big)
      throw Fail{NLFEM_GPU_BALL_EXITS_MESH,
                 "BallExitsMesh: ball reaches past an unglued facet of element " +
                     std::to_string(err_elem_h)};
    S.npairs = poff[S.phi];
  }
  // events of unit-buffer set k: units start / end, combine ready / done
  auto evu = [&](int set, int k) { return S.ev[14 + 4 * set + k]; };
  bool set_busy[2] = {false, false};   // a combine may still read the set
  bool set_timed[2] = {false, false};  // units events not yet accumulated
  auto collect = [&](int set) {        // Monte Carlo phase time of the set's last chunk
    if (!set_timed[set]) return;
    CK(cudaEventSynchronize(evu(set, 1)));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, evu(set, 0), evu(set, 1)));
    mc_ms += ms;
    set_timed[set] = false;
  };
  if (shard_hi > shard_lo) {
    int ii0 = shard_lo;
    int chunk = 0;
    while (ii0 < shard_hi) {
      int ii1;
      long long P0, np;
      if (fast) {
        ii1 = shard_hi;
        P0 = full_run ? 0 : S.installed_base;
        np = full_run ? S.survivors : S.shard_npairs;  // bound on the chunk's pairs
      } else {
        ii1 = (int)(std::upper_bound(poff.begin() + ii0 + 1, poff.begin() + shard_hi + 1,
                                     poff[ii0] + kPairsPerChunk) -
                    poff.begin()) - 1;
        ii1 = std::min(std::max(ii1, ii0 + 1), shard_hi);
        P0 = poff[ii0];
        np = poff[ii1] - P0;
      }
      if (probing) {  // overlap mode by measurement (see above)
        if (chunk == kProbe0 || chunk == kProbe0 + kProbeLen || chunk == kProbe0 + 2 * kProbeLen)
          CK(cudaEventRecord(S.ev[24 + (chunk - kProbe0) / kProbeLen], st));
        if (chunk == kProbe0) ov_bits = 3;
        if (chunk == kProbe0 + kProbeLen) ov_bits = 0;
        if (chunk == kProbe0 + 2 * kProbeLen + 2) {
          float with = 0, without = 0;
          CK(cudaEventSynchronize(S.ev[26]));
          CK(cudaEventElapsedTime(&with, S.ev[24], S.ev[25]));
          CK(cudaEventElapsedTime(&without, S.ev[25], S.ev[26]));
          ov_bits = with < 0.99f * without ? 3 : 0;
          if (std::getenv("NLFEM_GPU_TRACE"))
            fprintf(stderr, "[nlfem] overlap probe: %d chunks with %.2f ms, without %.2f ms -> %s\n",
                    kProbeLen, with, without, ov_bits ? "on" : "off");
        }
        overlap = ov_bits != 0;
      }
      const int set = chunk & 1;
      auto& U = S.ub[set];
      if (set_busy[set]) {  // the combine of chunk - 2 still reads this set
        CK(cudaStreamWaitEvent(st, evu(set, 3), 0));
        collect(set);
      }
      const long long* pend = S.pair_off.p + ii1;  // the chunk's actual pair end
      long long nitems = 0;
      if (need_units) {
        U.ucount.ensure(np + 1);
        U.uoff.ensure(np + 1);
        U.pair_outer.ensure(np + 1);
        k_units_count<<<nblk(np, 256), 256, 0, st>>>(P0, np, pend, S.info.p, U.ucount.p);
        k_pair_outer<<<nblk(32LL * (ii1 - ii0), 256), 256, 0, st>>>(ii0, ii1, S.pair_off.p, P0,
                                                                    U.pair_outer.p);
        S.launches += 2;
        U.nlist.ensure(16);  // 8 list lengths, 8 work cursors
        CK(cudaMemsetAsync(U.nlist.p, 0, 16 * sizeof(int), st));
        scan64(S, U.ucount.p, true, np, U.uoff.p, st);
        // buffers by the upper bound (4 items per pair): no count read-back
        nitems = 4 * np;
        U.mom.ensure(kMomStride * (size_t)(nitems + 1));
        U.ulist.ensure(8 * (size_t)(nitems + 1));
        k_units_fill<<<nblk(np, kFillThreads), kFillThreads, 0, st>>>(
            P0, np, pend, S.info.p, U.uoff.p, U.pair_outer.p, S.partner.p, U.ulist.p,
            nitems + 1, U.nlist.p);
        ++S.launches;
        CK(cudaEventRecord(evu(set, 0), st));
        cudaStream_t s3 = S.stream3;
        CK(cudaEventRecord(S.ev[10], st));  // fork
        CK(cudaStreamWaitEvent(s3, S.ev[10], 0));
        const long long ls = nitems + 1;
        // list lengths stay on the device: launches of two waves of resident CTAs
        int nl[8];
        for (int k = 0; k < 8; ++k)
          nl[k] = (int)std::min<long long>(nitems, (long long)S.sms * NLFEM_MC_MINBLOCKS * 2 * kMcThreads);
        // overlap mode: every units launch's shared memory is padded up to
        // kMcPadBytes in total, which caps the launch at three resident CTAs per
        // SM (48K registers) and leaves a quarter of the registers and ~54 KB of
        // shared memory for the co-resident combine CTA of the previous chunk
        // (once the combine's slot-map size is known, and only if its CTA then
        // fits beside three padded ones; otherwise the resident combine CTAs,
        // launched first, hold their registers and the units fit three beside
        // them anyway)
        const int mc_pad = (overlap && (ov_bits & 2) && combine_ready && fits_pad()) ? kMcPadBytes : 0;
        auto launch = [&](auto kern, int kind, cudaStream_t s) {
          if (nl[kind] <= 0) return;
          int dyn = 0;
          if (mc_pad > 0) {  // pad the launch's shared memory up to mc_pad bytes in total
            cudaFuncAttributes fa;
            CK(cudaFuncGetAttributes(&fa, kern));
            dyn = std::max(0, mc_pad - (int)fa.sharedSizeBytes);
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
          }
          if (overlap_able)  // see the combine's launch below
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    mc_pad > 0 ? (int)cudaSharedmemCarveoutMaxShared
                                               : (int)cudaSharedmemCarveoutDefault));
          kern<<<nblk(nl[kind], kMcThreads), kMcThreads, dyn, s>>>(
              P0, nitems, U.ulist.p + kind * ls, U.nlist.p + kind, U.mom.p, S.counters.p + 1);
          ++S.launches;
        };
        // lists 0..3: interior parents by cap case, 4..7: constraint parents;
        // the big straddle lists on `stream`, the rest beside them on s3
        if (need_mc) {
          launch(k_mc<false, false, 2>, 2, st);
          launch(k_mc<false, false, 1>, 1, st);
          launch(k_mc<false, false, 3>, 3, s3);
          launch(k_mc<false, false, 0>, 0, s3);
          if (S.g_deg <= 2) {
            launch(k_mc<true, true, 2>, 6, st);
            launch(k_mc<true, true, 1>, 5, st);
            launch(k_mc<true, true, 3>, 7, s3);
            launch(k_mc<true, true, 0>, 4, s3);
          } else {
            launch(k_mc<true, false, 2>, 6, st);
            launch(k_mc<true, false, 1>, 5, st);
            launch(k_mc<true, false, 3>, 7, s3);
            launch(k_mc<true, false, 0>, 4, s3);
          }
        } else if (D.strategy == NLFEM_STRATEGY_APPROXCAPS) {  // sphere-point hulls
          for (int kind : {1, 2, 3}) launch(k_approx<false>, kind, kind == 3 ? s3 : st);
          for (int kind : {5, 6, 7}) launch(k_approx<true>, kind, kind == 7 ? s3 : st);
        } else {  // nocaps: inner pieces only
          launch(k_mc<false, false, 2, false>, 2, st);
          launch(k_mc<false, false, 1, false>, 1, st);
          launch(k_mc<false, false, 3, false>, 3, s3);
          launch(k_mc<true, false, 2, false>, 6, st);
          launch(k_mc<true, false, 1, false>, 5, st);
          launch(k_mc<true, false, 3, false>, 7, s3);
        }
        CK(cudaEventRecord(S.ev[11], s3));  // join
        CK(cudaStreamWaitEvent(st, S.ev[11], 0));
        CK(cudaEventRecord(evu(set, 1), st));
        set_timed[set] = true;
      }
      setup_combine();
      // the combine of this chunk on stream4, after its units (and the
      // accumulator set-up) on `stream`; the next chunk's units proceed on
      // `stream` meanwhile
#ifndef NLFEM_COMB_SERIAL
#define NLFEM_COMB_SERIAL 0  // 1: the combine on `stream`, after its chunk's units
#endif
      cudaStream_t s4 = NLFEM_COMB_SERIAL ? st : S.stream4;
      CK(cudaEventRecord(evu(set, 2), st));
      CK(cudaStreamWaitEvent(s4, evu(set, 2), 0));
      // block size from delta/h (pairs per outer element grow like (delta/h)^3):
      // a property of the mesh, the same for every shard and chunk -- the
      // per-warp partial sums, hence the last bits, must not depend on sharding
#ifndef NLFEM_COMB_THREADS
#define NLFEM_COMB_THREADS 0  // 0: by delta/h; 128 / 256: forced
#endif
      // (Monte Carlo runs take 128 threads as well: their combine runs beside
      // the next chunk's units, below.)  Grid: one CTA per outer element, or --
      // overlap mode, every chunk but the last -- one resident CTA per SM
      // walking the chunk's elements while the next chunk's units, capped at
      // three CTAs per SM, use the rest of the SM
      const int nelem = ii1 - ii0;
      // (only if that CTA fits beside three units CTAs, padded or not)
      const bool resident = overlap && (ov_bits & 1) && (fits_pad() || fits_nopad()) && ii1 < shard_hi;
      if (chunk == 1 && std::getenv("NLFEM_GPU_TRACE"))
        fprintf(stderr, "[nlfem] combine: maxlen %d hcap %d ismem %zu overlap %d fits_pad %d "
                        "fits_nopad %d resident %d nelem %d\n", maxlen, hcap, ismem, (int)overlap,
                (int)fits_pad(), (int)fits_nopad(), (int)resident, ii1 - ii0);
      const int cgrid = resident ? 4 * S.sms : nelem;
      // The SM's shared-memory carve-out is set by the first kernel to land on
      // it: a resident combine CTA with a small slot map (24 KB at C4) left the SM
      // configured for ~100 KB, where only one 57-KB units CTA fitted beside it
      // until the SM drained (units 27% slower at C4).  In overlap mode both
      // kernels ask for the largest carve-out; otherwise the default (the
      // combine alone is 7% faster with its L1).
      if (overlap_able) {
        const int co = resident ? (int)cudaSharedmemCarveoutMaxShared
                                : (int)cudaSharedmemCarveoutDefault;
        CK(cudaFuncSetAttribute(k_integrate<128>, cudaFuncAttributePreferredSharedMemoryCarveout, co));
        CK(cudaFuncSetAttribute(k_integrate<256>, cudaFuncAttributePreferredSharedMemoryCarveout, co));
      }
      int* spread = nullptr;
      if (resident) {
        S.spread.ensure(1 + 1024);
        CK(cudaMemsetAsync(S.spread.p, 0, (1 + 1024) * sizeof(int), s4));
        spread = S.spread.p;
      }
      if (NLFEM_COMB_THREADS == 128 ||
          (NLFEM_COMB_THREADS == 0 && (need_mc || S.delta_over_h < 2.5)))
        k_integrate<128><<<cgrid, 128, ismem, s4>>>(
            ii0, S.pair_off.p, S.partner.p, S.info.p, S.soff.p, S.scols.p, S.eslot.p, S.V.p,
            S.rhsT.p, U.uoff.p, need_units ? U.mom.p : nullptr, P0, S.counters.p + 1, hcap,
            rowcap, nelem, spread);
      else
        k_integrate<256><<<cgrid, 256, ismem, s4>>>(
            ii0, S.pair_off.p, S.partner.p, S.info.p, S.soff.p, S.scols.p, S.eslot.p, S.V.p,
            S.rhsT.p, U.uoff.p, need_units ? U.mom.p : nullptr, P0, S.counters.p + 1, hcap,
            rowcap, nelem, spread);
      ++S.launches;
      CK(cudaEventRecord(evu(set, 3), s4));
      set_busy[set] = true;
      ii0 = ii1;
      ++chunk;
    }
  }
  // everything after the chunks (finalize, read-backs) waits for the combines
  for (int set = 0; set < 2; ++set) {
    if (set_busy[set]) CK(cudaStreamWaitEvent(st, evu(set, 3), 0));
    collect(set);
  }
  S.mc_ms = mc_ms;
  setup_combine();  // empty shard: the pattern is still needed by finalize
  CK(cudaEventRecord(S.ev[4], st));

  // ---- K6: finalize
  if (finalize) run_finalize(S, 0, S.unknowns);
  CK(cudaEventRecord(S.ev[5], st));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  unsigned long long cnt[9];
  CK(cudaMemcpy(cnt, S.counters.p, sizeof(cnt), cudaMemcpyDeviceToHost));
  if (npairs_pending) {  // deferred from the pairs phase (no round trip there)
    long long tot = 0;
    int e = big;
    CK(cudaMemcpy(&tot, S.pair_off.p + S.phi, sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&e, S.err_elem.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (e != big)
      throw Fail{NLFEM_GPU_BALL_EXITS_MESH,
                 "BallExitsMesh: ball reaches past an unglued facet of element " + std::to_string(e)};
    S.npairs = tot;
  }
  if (NLFEM_CHECKED) {
    const std::string g = guard_check();
    if (!g.empty()) throw Fail{NLFEM_GPU_ENODEVICE, "checked build: " + g};
  }
  S.items = cnt[0];
  S.mc_samples = cnt[1];
  S.mc_hits = cnt[2];
  S.ledger = cnt[3] + cnt[5];
  S.ledger_units = cnt[3];
  S.mc_subs = cnt[4];
  if (cnt[8])
    throw Fail{NLFEM_GPU_BAD_CONFIG,
               "BadConfig: the rows of an outer element's nodes outgrew the integration "
               "kernel's slot table (interaction neighbourhood too large)"};
  if (cnt[7])
    throw Fail{NLFEM_GPU_DEGENERATE_HULL,
               "DegenerateHull: approxcaps hull face table overflow (more than 32 faces)"};
  if (user) {
    CK(cudaEventRecord(S.ev[6], st));
    CK(cudaStreamWaitEvent(user, S.ev[6], 0));
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    float ms[6];
    for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&ms[i], S.ev[i], S.ev[i + 1]));
    // pattern: its own stream, overlapping the integrate phase (which is timed
    // from the end of the pairs phase)
    CK(cudaEventElapsedTime(&ms[2], S.ev[8], S.ev[9]));
    CK(cudaEventElapsedTime(&ms[5], S.ev[0], S.ev[5]));
    for (int i = 0; i < 5; ++i) stats->phase_ms[i] = ms[i];
    stats->device_ms = ms[5];
    stats->threads = 1;
    stats->blocks = (KI + 31) / 32;
    stats->mc_samples = S.mc_samples;
    stats->mc_hits = S.mc_hits;
    stats->element_pairs = S.npairs;
    {
      long long a = 0, b = 0;
      if (KI > 0) {
        CK(cudaMemcpy(&a, S.pair_off.p + shard_lo, sizeof(long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&b, S.pair_off.p + shard_hi, sizeof(long long), cudaMemcpyDeviceToHost));
      }
      stats->shard_pairs = b - a;
    }
    stats->items = (long long)S.items;
    stats->nnz_ext = S.nnz_s;
    stats->ledger_flops = S.ledger;
    stats->ledger_flops_units = S.ledger_units;
    stats->mc_subsimplices = S.mc_subs;
    stats->phase_ms[5] = S.mc_ms;
    stats->seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  }
}

int guard(char* err, size_t errlen, const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const Fail& f) {
    put_err(err, errlen, f.msg);
    return f.code;
  } catch (const std::bad_alloc&) {
    put_err(err, errlen, "out of host memory");
    return NLFEM_GPU_ENOMEM;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return NLFEM_GPU_ENODEVICE;
  }
}
}  // namespace

// ---------------------------------------------------------------------------
// solve_problem + l2_error (reference study.cpp:38-99) on the assembled system

// node values (study.cpp:64-74): unknowns from x, constrained nodes g(x_j);
// per-block maxima of |u_h(x_j) - exact(x_j)|
constexpr int kStudyThreads = 256;
__global__ void __launch_bounds__(kStudyThreads) k_node_values(int J, const double* node,
                                                               const int* dof, const double* x,
                                                               Poly g, Poly exact, double* vals,
                                                               double* bmax) {
  __shared__ double sm[kStudyThreads / 32];
  const int j = blockIdx.x * kStudyThreads + threadIdx.x;
  double e = 0;
  if (j < J) {
    const Vd p = {node[3 * j], node[3 * j + 1], node[3 * j + 2]};
    const int d = dof[j];
    const double v = d >= 0 ? x[d] : poly_eval(g, p);
    vals[j] = v;
    e = fabs(v - poly_eval(exact, p));
  }
  for (int sh = 16; sh > 0; sh >>= 1) e = fmax(e, __shfl_xor_sync(FULLMASK, e, sh));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0;
    for (int w = 0; w < kStudyThreads / 32; ++w) m = fmax(m, sm[w]);
    bmax[blockIdx.x] = m;
  }
}

// degree-5 14-point rule (reference quadrature.cpp:42-62): barycentric rows, weights
__constant__ double cL2Rule[14][5];

// per-block sums of vol_t w_q (u_h - exact)^2 over interior elements (thread
// per element, fixed order inside a block: warp tree, then warps in order)
__global__ void __launch_bounds__(kStudyThreads) k_l2_partial(int KI, const int* interior,
                                                              const int4* verts, const double* vol,
                                                              const double* node, const double* vals,
                                                              Poly exact, double* bsum) {
  __shared__ double sm[kStudyThreads / 32];
  const int i = blockIdx.x * kStudyThreads + threadIdx.x;
  double acc = 0;
  if (i < KI) {
    const int t = interior[i];
    const int4 w = verts[t];
    const int vv[4] = {w.x, w.y, w.z, w.w};
    Vd x[4];
    double u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[k] = {node[3 * vv[k]], node[3 * vv[k] + 1], node[3 * vv[k] + 2]};
      u[k] = vals[vv[k]];
    }
    const double V = vol[t];
    for (int q = 0; q < 14; ++q) {
      Vd p = {0.0, 0.0, 0.0};
      double uh = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double b = cL2Rule[q][k];
        p = vadd(p, vscale(b, x[k]));
        uh += b * u[k];
      }
      const double d = uh - poly_eval(exact, p);
      acc += V * cL2Rule[q][4] * d * d;
    }
  }
  for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, sh);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < kStudyThreads / 32; ++w) s += sm[w];
    bsum[blockIdx.x] = s;
  }
}

// one CTA: block sums in a fixed order -> sqrt; block maxima -> max
__global__ void __launch_bounds__(kStudyThreads) k_study_final(int nb_sum, const double* bsum,
                                                               int nb_max, const double* bmax,
                                                               double* res) {
  __shared__ double ss[kStudyThreads], sx[kStudyThreads];
  double a = 0, m = 0;
  for (int i = threadIdx.x; i < nb_sum; i += kStudyThreads) a += bsum[i];
  for (int i = threadIdx.x; i < nb_max; i += kStudyThreads) m = fmax(m, bmax[i]);
  ss[threadIdx.x] = a;
  sx[threadIdx.x] = m;
  __syncthreads();
  for (int h = kStudyThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      ss[threadIdx.x] += ss[threadIdx.x + h];
      sx[threadIdx.x] = fmax(sx[threadIdx.x], sx[threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    res[0] = sqrt(ss[0]);
    res[1] = sx[0];
  }
}

void session_solve(nlfem_gpu_session& S, double tol, int32_t max_iter, const nlfem_gpu_poly* exact,
                   double* u_node, nlfem_gpu_study* out) {
  if (S.nnz_out < 0 || !S.values.p)
    throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: solve needs an assembled system (run first)"};
  CK(cudaSetDevice(S.device));
  static std::atomic<unsigned long long> rule_set{0};  // bit d: uploaded to device d
  if (!(rule_set.load() >> (S.device & 63) & 1ull)) {
    const double a = 0.3108859192633005, wa = 0.1126879257180162;
    const double b = 0.0927352503108912, wb = 0.0734930431163619;
    const double c = 0.0455037041256497, d = 0.5 - c, wc = 0.0425460207770812;
    const double a4 = 1.0 - 3.0 * a, b4 = 1.0 - 3.0 * b;
    const double rows[14][5] = {{a4, a, a, a, wa}, {a, a4, a, a, wa}, {a, a, a4, a, wa},
                                {a, a, a, a4, wa}, {b4, b, b, b, wb}, {b, b4, b, b, wb},
                                {b, b, b4, b, wb}, {b, b, b, b4, wb}, {c, c, d, d, wc},
                                {c, d, c, d, wc}, {c, d, d, c, wc}, {d, c, c, d, wc},
                                {d, c, d, c, wc}, {d, d, c, c, wc}};
    CK(cudaMemcpyToSymbol(cL2Rule, rows, sizeof(rows)));
    rule_set.fetch_or(1ull << (S.device & 63));
  }
  Poly ex, g;
  poly_to_dev(exact, ex);
  g = S.dev.g;
  cudaStream_t st = S.stream;
  CK(cudaEventRecord(S.ev[12], st));
  S.solx.ensure(std::max(S.unknowns, 1));
  char cgerr[512] = {0};
  nlfem_gpu_solve_report rep{};
  const int rc = nlfem_gpu_cg_device(S.unknowns, reinterpret_cast<const int64_t*>(S.ooff.p), S.ocols.p, S.values.p, S.rhs.p, tol,
                                     max_iter, S.solx.p, st, &rep, cgerr, sizeof(cgerr));
  if (rc) throw Fail{rc, cgerr};
  const int nbJ = std::max(1, (S.J + kStudyThreads - 1) / kStudyThreads);
  const int nbK = std::max(1, (S.KI + kStudyThreads - 1) / kStudyThreads);
  S.nodev.ensure(std::max(S.J, 1));
  S.study_tmp.ensure(nbJ + nbK + 2);
  double* bmax = S.study_tmp.p;
  double* bsum = bmax + nbJ;
  double* res = bsum + nbK;
  if (S.J > 0)
    k_node_values<<<nbJ, kStudyThreads, 0, st>>>(S.J, S.node.p, S.dof.p, S.solx.p, g, ex,
                                                 S.nodev.p, bmax);
  else
    CK(cudaMemsetAsync(bmax, 0, sizeof(double), st));
  if (S.KI > 0)
    k_l2_partial<<<nbK, kStudyThreads, 0, st>>>(S.KI, S.interior.p, S.verts.p, S.vol.p, S.node.p,
                                                S.nodev.p, ex, bsum);
  else
    CK(cudaMemsetAsync(bsum, 0, sizeof(double), st));
  k_study_final<<<1, kStudyThreads, 0, st>>>(S.KI > 0 ? nbK : 1, bsum, S.J > 0 ? nbJ : 1, bmax,
                                             res);
  CK(cudaGetLastError());
  CK(cudaEventRecord(S.ev[13], st));
  double h[2];
  CK(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (u_node && S.J > 0)
    CK(cudaMemcpyAsync(u_node, S.nodev.p, sizeof(double) * S.J, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, S.ev[12], S.ev[13]));
  out->iterations = rep.iterations;
  out->converged = rep.converged;
  out->relative_residual = rep.relative_residual;
  out->l2_error = h[0];
  out->max_nodal_error = h[1];
  out->device_ms = ms;
}

// Every entry point that touches a session runs under its device's lock and
// with that device current (the caller's current device is restored on
// return).  Sessions on one device share the per-device __constant__
// parameter block cD, which each run / finalize rebinds, so two host threads
// (ctypes releases the GIL) or two sessions driven alternately must not
// interleave on a device.  Recursive: the one-shot call nests session calls.
std::recursive_mutex& device_mutex(int dev) {
  static std::recursive_mutex mu[64];
  return mu[dev & 63];
}
struct DeviceScope {
  int prev = -1;
  std::unique_lock<std::recursive_mutex> lk;
  explicit DeviceScope(int dev) : lk(device_mutex(dev < 0 ? 0 : dev)) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && prev != dev) cudaSetDevice(dev);  // a failure surfaces at the next CK
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
int config_device(const nlfem_gpu_config* cfg) {
  int dev = cfg ? cfg->device : -1;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

__global__ void k_guard_poke(int* a, long long i) { a[i] = 7; }

extern "C" {

// Checked builds only: proves the canaries catch an out-of-bounds write (a
// kernel writes one element past a fresh buffer).  Returns 1 if caught, 0 if
// not, -1 in the default build.
int nlfem_gpu_debug_guard_selftest(int32_t past) {
  if (!NLFEM_CHECKED) return -1;
  try {
    DBuf<int> b;
    b.ensure(1000);
    k_guard_poke<<<1, 1>>>(b.p, past ? 1000 : 999);
    CK(cudaDeviceSynchronize());
    const std::string g = guard_check();
    return g.empty() ? 0 : 1;
  } catch (...) {
    return -2;
  }
}

int nlfem_gpu_fp64_peak(int32_t device, double* tflops, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    if (device >= 0) CK(cudaSetDevice(device));
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<double> out;
    out.ensure(1);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int iters = 1 << 14, blocks = sms * 8, threads = 256;
    k_dfma_peak<<<blocks, threads>>>(out.p, 256, 0.999999, 1e-7);  // warm-up
    CK(cudaEventRecord(e0));
    k_dfma_peak<<<blocks, threads>>>(out.p, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

const char* nlfem_gpu_version(void) { return "nlfem_gpu 0.2 sm_100a (inside, overlap, barycenter, nocaps, approxcaps, fullcaps)"; }

int nlfem_gpu_session_create(const nlfem_gpu_mesh* mesh, const nlfem_gpu_dofs* dofs,
                             const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                             const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                             nlfem_gpu_session** out, char* err, size_t errlen) {
  *out = nullptr;
  auto* S = new nlfem_gpu_session;
  const int rc = guard(err, errlen, [&] {
    DeviceScope ds(config_device(cfg));
    session_init(*S, mesh, dofs, kernel, f, g, cfg);
  });
  if (rc) {
    nlfem_gpu_session_destroy(S);
    return rc;
  }
  *out = S;
  return 0;
}

int nlfem_gpu_session_reset(nlfem_gpu_session* s, const nlfem_gpu_mesh* mesh,
                            const nlfem_gpu_dofs* dofs, const nlfem_gpu_kernel* kernel,
                            const nlfem_gpu_poly* f, const nlfem_gpu_poly* g,
                            const nlfem_gpu_config* cfg, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(config_device(cfg));
    s->pairs_installed = false;
    session_init(*s, mesh, dofs, kernel, f, g, cfg);
  });
}

int nlfem_gpu_session_run(nlfem_gpu_session* s, void* stream, nlfem_gpu_stats* stats, char* err,
                          size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    run_all(*s, static_cast<cudaStream_t>(stream), stats, 0, s->KI, true);
  });
}

int nlfem_gpu_session_run_shard(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                int32_t finalize, nlfem_gpu_stats* stats, char* err,
                                size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    run_all(*s, static_cast<cudaStream_t>(stream), stats, lo, hi, finalize != 0);
  });
}

int nlfem_gpu_session_run_local(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                nlfem_gpu_stats* stats, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    s->pairs_installed = false;
    run_all(*s, static_cast<cudaStream_t>(stream), stats, lo, hi, false, true);
  });
}

int nlfem_gpu_session_halo_records(nlfem_gpu_session* s, int32_t world, const int32_t* bounds,
                                   void** keys, void** vals, int64_t* counts, char* err,
                                   size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    nlfem_gpu_session& S = *s;
    cudaStream_t st = S.stream;
    if (world < 1 || world > 64 || bounds[0] != 0 || bounds[world] != S.unknowns)
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: row bounds must split [0, unknowns) in <= 64 blocks"};
    const int U = S.unknowns;
    CK(cudaMemcpyToSymbolAsync(cD, &S.dev, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
    S.hcnt.ensure(U + 1);
    S.hoff.ensure(U + 1);
    if (U > 0) {
      k_halo_count<<<nblk(U, 256), 256, 0, st>>>(S.soff.p, S.dof_node.p, S.hcnt.p);
      ++S.launches;
    }
    scan64(S, S.hcnt.p, true, U, S.hoff.p, st);
    std::vector<long long> off(U + 1, 0);
    CK(cudaMemcpyAsync(off.data(), S.hoff.p, sizeof(long long) * (U + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const long long n = off[U];
    S.hkeys.ensure(n + 1);
    S.hvals.ensure(4 * (n + 1));
    if (U > 0 && n > 0) {
      k_halo_fill<<<nblk(32LL * U, 256), 256, 0, st>>>(S.soff.p, S.scols.p, S.mirror.p, S.V.p,
                                                       S.dof_node.p, S.hoff.p, S.hkeys.p, S.hvals.p);
      ++S.launches;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    for (int r = 0; r < world; ++r) counts[r] = off[bounds[r + 1]] - off[bounds[r]];
    *keys = S.hkeys.p;
    *vals = S.hvals.p;
  });
}

int nlfem_gpu_session_rhs_records(nlfem_gpu_session* s, int32_t world, const int32_t* bounds,
                                  void** idx, void** vals, int64_t* counts, char* err,
                                  size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    nlfem_gpu_session& S = *s;
    cudaStream_t st = S.stream;
    if (world < 1 || world > 64 || bounds[0] != 0 || bounds[world] != S.unknowns)
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: row bounds must split [0, unknowns) in <= 64 blocks"};
    CK(cudaMemcpyToSymbolAsync(cD, &S.dev, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
    const int n = S.phi - S.plo;
    DBuf<int> db;
    db.upload(bounds, world + 1, st);
    S.rmask.ensure(n + 1);
    S.rflag.ensure(n + 1);
    S.roffs.ensure(n + 1);
    if (n > 0) {
      k_rhs_mask<<<nblk(n, 256), 256, 0, st>>>(S.plo, S.phi, db.p, world, S.rmask.p);
      ++S.launches;
    }
    // per destination: flag, scan, count (a few host reads; world is small)
    std::vector<long long> cnt(world, 0);
    for (int r = 0; r < world; ++r) {
      if (n > 0) {
        k_rhs_flag<<<nblk(n, 256), 256, 0, st>>>(n, S.rmask.p, r, S.rflag.p);
        ++S.launches;
      }
      scan64(S, S.rflag.p, true, n, S.roffs.p, st);
      cnt[r] = read_ll(S.roffs.p + n, st);
    }
    long long tot = 0;
    for (int r = 0; r < world; ++r) tot += cnt[r];
    S.ridx.ensure(tot + 1);
    S.rvals.ensure((tot + 1) * (4 * kRhsWarps));
    long long base = 0;
    for (int r = 0; r < world; ++r) {
      if (cnt[r] > 0) {
        k_rhs_flag<<<nblk(n, 256), 256, 0, st>>>(n, S.rmask.p, r, S.rflag.p);
        scan64(S, S.rflag.p, true, n, S.roffs.p, st);
        k_rhs_scatter<<<nblk(n, 256), 256, 0, st>>>(n, S.plo, S.rflag.p, S.roffs.p, base, S.rhsT.p,
                                                    S.ridx.p, S.rvals.p);
        S.launches += 2;
      }
      counts[r] = cnt[r];
      base += cnt[r];
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    *idx = S.ridx.p;
    *vals = S.rvals.p;
  });
}

int nlfem_gpu_session_finalize_merged(nlfem_gpu_session* s, void* stream, int32_t row_lo,
                                      int32_t row_hi, const void* keys, const void* vals,
                                      int64_t n, const void* ridx, const void* rvals, int64_t m,
                                      char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    nlfem_gpu_session& S = *s;
    cudaStream_t st = S.stream;
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    if (user) {
      CK(cudaEventRecord(S.ev[7], user));
      CK(cudaStreamWaitEvent(st, S.ev[7], 0));
    }
    if (n < 0 || n >= (1LL << 32) - 1)
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: too many slot records for one rank"};
    CK(cudaMemcpyToSymbolAsync(cD, &S.dev, sizeof(Dev), 0, cudaMemcpyHostToDevice, st));
    const int J = S.J, U = S.unknowns;
    const int r0 = std::max(0, row_lo), r1 = std::max(r0, std::min(row_hi, U));
    // rhsT rows of the outer elements at this rank's nodes
    if (m > 0) {
      k_rhs_install<<<nblk(m * (4 * kRhsWarps), 256), 256, 0, st>>>(
          m, static_cast<const int*>(ridx), static_cast<const double*>(rvals), S.rhsT.p);
      ++S.launches;
    }
    // sort the records by key; distinct keys with their integer sums
    S.mkeys.ensure(n + 1);
    S.midx.ensure(n + 1);
    S.midx2.ensure(n + 1);
    S.mflag.ensure(n + 1);
    S.muid.ensure(n + 2);
    long long nu = 0;
    if (n > 0) {
      k_iota<<<nblk(n, 256), 256, 0, st>>>(n, S.midx.p);
      int endbit = 33;
      while (endbit < 64 && (1LL << (endbit - 32)) < (long long)J) ++endbit;
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, static_cast<const unsigned long long*>(keys),
                                         S.mkeys.p, S.midx.p, S.midx2.p, n, 0, endbit, st));
      S.cub_tmp.ensure(tb);
      CK(cub::DeviceRadixSort::SortPairs(S.cub_tmp.p, tb, static_cast<const unsigned long long*>(keys),
                                         S.mkeys.p, S.midx.p, S.midx2.p, n, 0, endbit, st));
      k_key_flag<<<nblk(n, 256), 256, 0, st>>>(n, S.mkeys.p, S.mflag.p);
      S.launches += 2;
      scan64(S, S.mflag.p, true, n, S.muid.p, st);
      nu = read_ll(S.muid.p + n, st);
    }
    DBuf<long long>& start = S.mstart;
    start.ensure(nu + 1);
    S.mV.ensure(4 * (size_t)(nu + 1));
    S.mcols.ensure(nu + 1);
    S.mmirror.ensure(nu + 1);
    S.mcnt.ensure(J + 1);
    CK(cudaMemsetAsync(S.mcnt.p, 0, (J + 1) * sizeof(int), st));
    if (n > 0) {
      k_key_start<<<nblk(n, 256), 256, 0, st>>>(n, S.mflag.p, S.muid.p, start.p);
      k_key_sum<<<nblk(nu, 256), 256, 0, st>>>(nu, start.p, S.mkeys.p, S.midx2.p, static_cast<const long long*>(vals),
                                               S.mV.p, S.mcols.p, S.mmirror.p, S.mcnt.p);
      S.launches += 2;
    }
    S.moff.ensure(J + 1);
    scan64(S, S.mcnt.p, true, J, S.moff.p, st);
    // output pattern and values of the row block from the merged rows
    CK(cudaMemsetAsync(S.ovf.p, 0, sizeof(int), st));
    S.olen.ensure(U);
    S.ooff.ensure(U + 1);
    k_outpat<false><<<nblk(32LL * U, 256), 256, 0, st>>>(S.moff.p, S.mcols.p, S.olen.p, nullptr,
                                                         nullptr, nullptr, S.dof_node.p, S.ovf.p);
    scan64(S, S.olen.p, true, U, S.ooff.p, st);
    const long long nnz = read_ll(S.ooff.p + U, st);
    S.ocols.ensure(nnz + 1);
    S.omap.ensure(nnz + 1);
    k_outpat<true><<<nblk(32LL * U, 256), 256, 0, st>>>(S.moff.p, S.mcols.p, nullptr, S.ooff.p,
                                                        S.ocols.p, S.omap.p, S.dof_node.p, S.ovf.p);
    S.nnz_out = nnz;
    S.values.ensure(nnz + 1);
    S.rhs.ensure(U + 1);
    if (r1 > r0) {
      k_finalize<<<nblk((long long)(r1 - r0) * 32, 128), 128, 0, st>>>(
          S.moff.p, S.mcols.p, S.mmirror.p, S.mV.p, S.ooff.p, S.omap.p, S.values.p, S.rhsT.p,
          S.rhs.p, S.dof_node.p, r0, r1);
      ++S.launches;
    }
    S.launches += 2;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    if (NLFEM_CHECKED) {
      const std::string g = guard_check();
      if (!g.empty()) throw Fail{NLFEM_GPU_ENODEVICE, "checked build: " + g};
    }
    if (user) {
      CK(cudaEventRecord(S.ev[6], st));
      CK(cudaStreamWaitEvent(user, S.ev[6], 0));
    }
  });
}

int nlfem_gpu_session_pairs_shard(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                  int64_t* npairs, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    nlfem_gpu_session& S = *s;
    cudaStream_t st = S.stream;
    if (stream) {
      CK(cudaEventRecord(S.ev[7], static_cast<cudaStream_t>(stream)));
      CK(cudaStreamWaitEvent(st, S.ev[7], 0));
    }
    lo = std::max(0, std::min(lo, S.KI));
    hi = std::max(lo, std::min(hi, S.KI));
    S.launches = 0;
    S.pairs_installed = false;
    run_prep(S);
    build_pairs(S, lo, hi);
    long long tot = 0;
    int e = 0;
    CK(cudaMemcpyAsync(&tot, S.pair_off.p + hi, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&e, S.err_elem.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (e != 0x7fffffff)
      throw Fail{NLFEM_GPU_BALL_EXITS_MESH,
                 "BallExitsMesh: ball reaches past an unglued facet of element " + std::to_string(e)};
    S.pairs_lo = lo;
    S.pairs_hi = hi;
    S.shard_npairs = tot;
    if (npairs) *npairs = tot;
  });
}

int nlfem_gpu_session_pairs_shard_out(nlfem_gpu_session* s, void** counts, void** partners,
                                      int64_t* npairs) {
  *counts = s->pair_count.p + s->pairs_lo;
  *partners = s->partner.p;
  *npairs = s->shard_npairs;
  return 0;
}

int nlfem_gpu_session_pairs_install(nlfem_gpu_session* s, void* stream, const void* counts,
                                    const void* partners, int64_t npairs_total, char* err,
                                    size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    nlfem_gpu_session& S = *s;
    cudaStream_t st = S.stream;
    if (stream) {
      CK(cudaEventRecord(S.ev[7], static_cast<cudaStream_t>(stream)));
      CK(cudaStreamWaitEvent(st, S.ev[7], 0));
    }
    const int KI = S.KI;
    // keep this rank's own codes, then the global counts, offsets and partners
    S.info_own.ensure(S.shard_npairs + 1);
    if (S.shard_npairs)
      CK(cudaMemcpyAsync(S.info_own.p, S.info.p, S.shard_npairs * sizeof(unsigned),
                         cudaMemcpyDeviceToDevice, st));
    if (counts != S.pair_count.p)
      CK(cudaMemcpyAsync(S.pair_count.p, counts, (size_t)KI * sizeof(int),
                         cudaMemcpyDeviceToDevice, st));
    scan64(S, S.pair_count.p, true, KI, S.pair_off.p, st);
    long long base = 0, tot = 0;
    CK(cudaMemcpyAsync(&base, S.pair_off.p + S.pairs_lo, sizeof(long long), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaMemcpyAsync(&tot, S.pair_off.p + KI, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (tot != npairs_total)
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: installed pair counts do not add up"};
    S.installed_base = base;
    S.npairs = tot;
    S.partner.ensure(std::max<long long>(1, tot));
    S.info.ensure(std::max<long long>(1, tot));
    if (tot && partners != S.partner.p)
      CK(cudaMemcpyAsync(S.partner.p, partners, tot * sizeof(int), cudaMemcpyDeviceToDevice, st));
    // codes are needed only for this rank's outer elements; the rest stay zero
    if (tot) CK(cudaMemsetAsync(S.info.p, 0, tot * sizeof(unsigned), st));
    if (S.shard_npairs)
      CK(cudaMemcpyAsync(S.info.p + base, S.info_own.p, S.shard_npairs * sizeof(unsigned),
                         cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    S.pairs_installed = true;
  });
}

int nlfem_gpu_session_partials(nlfem_gpu_session* s, void** V, int64_t* nwords, void** rhsT,
                               int64_t* nrhs) {
  *V = s->V.p;
  *nwords = 2 * s->nnz_s;
  *rhsT = s->rhsT.p;
  *nrhs = 4 * kRhsWarps * (int64_t)s->KI;
  return 0;
}

int nlfem_gpu_session_solve(nlfem_gpu_session* s, double tol, int32_t max_iter,
                            const nlfem_gpu_poly* exact, double* u_node, nlfem_gpu_study* out,
                            char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    session_solve(*s, tol, max_iter, exact, u_node, out);
  });
}

int nlfem_gpu_session_outputs(nlfem_gpu_session* s, void** row_off, void** col_idx,
                              void** values, void** rhs, int32_t* rows, int64_t* nnz) {
  *row_off = s->ooff.p;
  *col_idx = s->ocols.p;
  *values = s->values.p;
  *rhs = s->rhs.p;
  *rows = s->unknowns;
  *nnz = s->nnz_out;
  return 0;
}

int nlfem_gpu_session_finalize(nlfem_gpu_session* s, void* stream, int32_t row_lo,
                               int32_t row_hi, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    if (user) {
      CK(cudaEventRecord(s->ev[7], user));
      CK(cudaStreamWaitEvent(s->stream, s->ev[7], 0));
    }
    CK(cudaMemcpyToSymbolAsync(cD, &s->dev, sizeof(Dev), 0, cudaMemcpyHostToDevice, s->stream));
    run_finalize(*s, std::max(0, row_lo), std::min(row_hi, s->unknowns));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));
  });
}

int nlfem_gpu_session_download_rows(nlfem_gpu_session* s, int32_t row_lo, int32_t row_hi,
                                    nlfem_gpu_csr* out, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    const int r0 = std::max(0, row_lo), r1 = std::max(r0, std::min(row_hi, s->unknowns));
    const int n = r1 - r0;
    std::vector<long long> off(n + 1);
    CK(cudaMemcpy(off.data(), s->ooff.p + r0, sizeof(long long) * (n + 1), cudaMemcpyDeviceToHost));
    const long long nnz = off[n] - off[0];
    out->rows = n;
    out->nnz = nnz;
    out->row_ptr = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (n + 1)));
    out->col_idx = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<long long>(nnz, 1)));
    out->values = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(nnz, 1)));
    out->rhs = static_cast<double*>(std::malloc(sizeof(double) * std::max(n, 1)));
    if (!out->row_ptr || !out->col_idx || !out->values || !out->rhs)
      throw Fail{NLFEM_GPU_ENOMEM, "out of host memory"};
    for (int i = 0; i <= n; ++i) out->row_ptr[i] = (int32_t)(off[i] - off[0]);
    if (nnz) {
      CK(cudaMemcpy(out->col_idx, s->ocols.p + off[0], sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(out->values, s->values.p + off[0], sizeof(double) * nnz, cudaMemcpyDeviceToHost));
    }
    if (n) CK(cudaMemcpy(out->rhs, s->rhs.p + r0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  });
}

int nlfem_gpu_session_download(nlfem_gpu_session* s, nlfem_gpu_csr* out, char* err,
                               size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    const int U = s->unknowns;
    const long long nnz = s->nnz_out;
    if (nnz > (long long)0x7fffffff)
      throw Fail{NLFEM_GPU_BAD_CONFIG, "BadConfig: nnz exceeds int32 row pointers"};
    // one page-locked block from the result pool: row_ptr | col_idx | values | rhs
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t br = al(4 * (size_t)(U + 1)), bc = al(4 * (size_t)nnz), bv = al(8 * (size_t)nnz);
    char* blk = g_result_pool.acquire(br + bc + bv + 8 * (size_t)std::max(U, 1));
    out->rows = U;
    out->nnz = nnz;
    out->row_ptr = reinterpret_cast<int32_t*>(blk);
    out->col_idx = reinterpret_cast<int32_t*>(blk + br);
    out->values = reinterpret_cast<double*>(blk + br + bc);
    out->rhs = reinterpret_cast<double*>(blk + br + bc + bv);
    // int32 row pointers on the device, then straight DMA into the result
    cudaStream_t st = s->stream;
    s->rowptr32.ensure(U + 1);
    k_ll_to_int<<<nblk(U + 1, 256), 256, 0, st>>>(U + 1, s->ooff.p, s->rowptr32.p);
    CK(cudaMemcpyAsync(out->row_ptr, s->rowptr32.p, 4 * (size_t)(U + 1), cudaMemcpyDeviceToHost, st));
    if (nnz) {
      CK(cudaMemcpyAsync(out->col_idx, s->ocols.p, 4 * (size_t)nnz, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(out->values, s->values.p, 8 * (size_t)nnz, cudaMemcpyDeviceToHost, st));
    }
    if (U) CK(cudaMemcpyAsync(out->rhs, s->rhs.p, 8 * (size_t)U, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int nlfem_gpu_session_pairs_device(nlfem_gpu_session* s, int64_t* npairs,
                                   const int64_t** outer_offsets, const int32_t** partner,
                                   const uint32_t** info) {
  *npairs = s->npairs;
  *outer_offsets = reinterpret_cast<const int64_t*>(s->pair_off.p);
  *partner = s->partner.p;
  *info = s->info.p;
  return 0;
}

int nlfem_gpu_session_pairs(nlfem_gpu_session* s, int64_t* npairs, int64_t* outer_offsets,
                            int32_t* partner, uint32_t* info, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    DeviceScope ds(s->device);
    *npairs = s->npairs;
    if (!outer_offsets) return;
    std::vector<long long> off(s->KI + 1);
    CK(cudaMemcpy(off.data(), s->pair_off.p, sizeof(long long) * (s->KI + 1), cudaMemcpyDeviceToHost));
    for (int i = 0; i <= s->KI; ++i) outer_offsets[i] = off[i];
    if (s->npairs) {
      CK(cudaMemcpy(partner, s->partner.p, sizeof(int32_t) * s->npairs, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(info, s->info.p, sizeof(uint32_t) * s->npairs, cudaMemcpyDeviceToHost));
    }
  });
}

int64_t nlfem_gpu_session_launches(const nlfem_gpu_session* s) { return s ? s->launches.load() : 0; }

void nlfem_gpu_session_destroy(nlfem_gpu_session* s) {
  if (!s) return;
  {
  DeviceScope ds(s->device);
  for (auto e : s->ev) cudaEventDestroy(e);
  if (s->stream) cudaStreamDestroy(s->stream);
  if (s->stream2) cudaStreamDestroy(s->stream2);
  if (s->stream3) cudaStreamDestroy(s->stream3);
  if (s->stream4) cudaStreamDestroy(s->stream4);
  }
  delete s;
}

// The one-shot entry keeps one workspace per device (stream, events, device
// buffers; grow-only) across calls, so repeated assemblies do not pay for
// cudaMalloc / cudaFree.  Calls from several host threads are serialised per
// device (the workspace and the device's parameter block are shared), so the
// entry is reentrant like the reference's pure assemble().
int nlfem_gpu_assemble(const nlfem_gpu_mesh* mesh, const nlfem_gpu_dofs* dofs,
                       const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                       const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                       nlfem_gpu_csr* out, nlfem_gpu_stats* stats, char* err, size_t errlen) {
  const auto t0 = std::chrono::steady_clock::now();
  static nlfem_gpu_session* workspaces[64] = {};
  const int dev = config_device(cfg);
  if (dev < 0 || dev >= 64) {
    std::snprintf(err, errlen, "BadConfig: device ordinal out of range");
    return NLFEM_GPU_BAD_CONFIG;
  }
  std::unique_lock<std::recursive_mutex> lk(device_mutex(dev));  // held to the download
  if (!workspaces[dev]) workspaces[dev] = new nlfem_gpu_session;
  nlfem_gpu_session* s = workspaces[dev];
  int rc = guard(err, errlen, [&] {
    DeviceScope ds(dev);
    session_init(*s, mesh, dofs, kernel, f, g, cfg);
  });
  if (rc) return rc;
  const auto t1 = std::chrono::steady_clock::now();
  rc = nlfem_gpu_session_run(s, nullptr, stats, err, errlen);
  const auto t2 = std::chrono::steady_clock::now();
  if (!rc) rc = nlfem_gpu_session_download(s, out, err, errlen);
  const auto t3 = std::chrono::steady_clock::now();
  if (!rc && stats)
    stats->seconds = std::chrono::duration<double>(t3 - t0).count();
  static const bool trace = std::getenv("NLFEM_GPU_TRACE") != nullptr;
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "nlfem_gpu_assemble: init %.3f ms, run %.3f ms, download %.3f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return rc;
}

void nlfem_gpu_free_csr(nlfem_gpu_csr* csr) {
  if (!csr) return;
  if (!csr->row_ptr || !g_result_pool.release(csr->row_ptr)) {  // pooled block, else malloc'd
    std::free(csr->row_ptr);
    std::free(csr->col_idx);
    std::free(csr->values);
    std::free(csr->rhs);
  }
  csr->row_ptr = csr->col_idx = nullptr;
  csr->values = csr->rhs = nullptr;
}

}  // extern "C"
