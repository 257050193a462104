// nlfem_setup.cu -- the reference's upstream setup (build_cmap +
// build_element_table + build_dofmap) on the GPU.
//
// Produces exactly the arrays of nlfem_host_element_table / nlfem_host_dofmap
// (host_setup.cpp), i.e. the reference's ElementTable and DofMap:
//   * validation (reference cmap.cpp:66-83): the first offending cell in
//     (cell, slot) order is found with one atomicMin over an order key, so the
//     error message names the same cell and vertex as the host;
//   * facet gluing (cmap.cpp:85-105): a node -> cell incidence list (CSR), then
//     one thread per (cell, facet) scans the cells of the facet's lowest-degree
//     vertex for the other cells holding all three vertices -- no sort; three or
//     more cells on one facet is NonManifold;
//   * orientation (cmap.cpp:107-140): the host BFS flips a cell iff its facet
//     orientations disagree with its component's lowest-id cell along any
//     path.  Here every cell holds (label << 1 | parity) -- "my flip relative
//     to cell label" -- and repeated relaxation over glued facets plus pointer
//     jumping (label of my label) drives it to (lowest id of the component,
//     flip); every value written is a true path relation, so at the fixpoint a
//     glued facet with inconsistent parities exists iff the mesh is not
//     orientable;
//   * per-element fields (ball_approx.cpp:51-95): FMA-free (-fmad=false), the
//     host's operation order, correctly rounded sqrt and division -> the same
//     bits as the host/reference;
//   * dof map (dofmap.cpp): constrained = vertex of any region cell; dof ids
//     by an exclusive scan in node order.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "nlfem_gpu.h"

namespace {

struct SetupFail {
  int code;
  std::string msg;
};

#define CKS(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw SetupFail{e_ == cudaErrorMemoryAllocation ? NLFEM_GPU_ENOMEM                \
                                                      : NLFEM_GPU_ENODEVICE,            \
                      std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x}; \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  void alloc(long long n) { CKS(cudaMalloc(&p, sizeof(T) * std::max<long long>(n, 1))); }
  ~DBuf() { cudaFree(p); }
};

constexpr int kThr = 256;
inline unsigned blocks(long long n) { return unsigned((n + kThr - 1) / kThr); }

__device__ __forceinline__ int parity3(int a, int b, int c) {
  return ((a > b) + (a > c) + (b > c)) & 1;
}

// (cell, slot) order key of the first failing check: slot i's range check
// precedes its repeat checks, as in the host loop.
__global__ void k_validate(const int4* cells, long long K, long long V, unsigned* deg,
                           unsigned long long* bad) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int4 c = cells[k];
  const int v[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (v[i] < 0 || v[i] >= V) {
      atomicMin(bad, (unsigned long long)k * 8 + i * 2);
      return;
    }
#pragma unroll
    for (int j = i + 1; j < 4; ++j)
      if (v[j] == v[i]) {
        atomicMin(bad, (unsigned long long)k * 8 + i * 2 + 1);
        return;
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) atomicAdd(&deg[v[i]], 1u);
}

__global__ void k_dangling(const unsigned* deg, long long V, unsigned long long* first) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V && deg[v] == 0) atomicMin(first, (unsigned long long)v);
}

__global__ void k_widen(const unsigned* deg, long long V, long long* off) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V) off[v] = deg[v];
}

__global__ void k_incidence(const int4* cells, long long K, const long long* off, unsigned* cur,
                            int* inc) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int4 c = cells[k];
  const int v[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) inc[off[v[i]] + atomicAdd(&cur[v[i]], 1u)] = (int)k;
}

// other[4k+s]: the cell across the facet opposite input slot s of cell k (-1:
// unglued); psum[4k+s]: XOR of the two cells' facet orientation parities.
__global__ void k_match(const int4* cells, long long K, const long long* off, const int* inc,
                        int* other, unsigned char* psum, int* nonmanifold) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= 4 * K) return;
  const long long k = f >> 2;
  const int s = int(f & 3);
  const int4 c = cells[k];
  const int v[4] = {c.x, c.y, c.z, c.w};
  int t[3], m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i != s) t[m++] = v[i];
  const int par = parity3(t[0], t[1], t[2]) ^ (s & 1);
  // scan the incidence list of the facet vertex with the fewest cells
  int a = 0;
  long long best = off[t[0] + 1] - off[t[0]];
#pragma unroll
  for (int i = 1; i < 3; ++i) {
    const long long d = off[t[i] + 1] - off[t[i]];
    if (d < best) best = d, a = i;
  }
  const int b = t[a == 0 ? 1 : 0], e = t[a == 2 ? 1 : 2];
  int cnt = 0, mo = -1, ms = 0;
  for (long long p = off[t[a]], pe = off[t[a] + 1]; p < pe; ++p) {
    const int mc = inc[p];
    if (mc == (int)k) continue;
    const int4 w4 = cells[mc];
    const int w[4] = {w4.x, w4.y, w4.z, w4.w};
    bool hb = false, he = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) hb |= w[i] == b, he |= w[i] == e;
    if (!(hb && he)) continue;
    ++cnt;
    mo = mc;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (w[i] != t[0] && w[i] != t[1] && w[i] != t[2]) ms = i;
  }
  if (cnt > 1) atomicOr(nonmanifold, 1);
  if (cnt == 1) {
    const int4 w4 = cells[mo];
    const int w[4] = {w4.x, w4.y, w4.z, w4.w};
    int u[3], n = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i != ms) u[n++] = w[i];
    other[f] = mo;
    psum[f] = (unsigned char)(par ^ parity3(u[0], u[1], u[2]) ^ (ms & 1));
  } else {
    other[f] = -1;
    psum[f] = 0;
  }
}

__global__ void k_label_init(long long K, unsigned long long* L) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < K) L[t] = (unsigned long long)t << 1;
}

// One relaxation sweep: my relation via each glued neighbour (its flip
// relative to its label, XOR the facet parity, XOR 1: adjacent cells must
// induce opposite orientations), then via my label's own relation.
__global__ void k_label_relax(long long K, const int4* other, const uchar4* psum,
                              unsigned long long* L, int* changed) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const unsigned long long cur = L[t];
  unsigned long long best = cur;
  const int4 o4 = other[t];
  const uchar4 p4 = psum[t];
  const int o[4] = {o4.x, o4.y, o4.z, o4.w};
  const unsigned ps[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (o[s] < 0) continue;
    const unsigned long long lo = L[o[s]];
    best = min(best, (lo & ~1ull) | ((lo ^ ps[s] ^ 1u) & 1ull));
  }
  const unsigned long long ll = L[best >> 1];
  best = min(best, (ll & ~1ull) | ((ll ^ best) & 1ull));
  if (best < cur) {
    L[t] = best;
    *changed = 1;
  }
}

__global__ void k_label_check(long long K, const int4* other, const uchar4* psum,
                              const unsigned long long* L, int* bad) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const int4 o4 = other[t];
  const uchar4 p4 = psum[t];
  const int o[4] = {o4.x, o4.y, o4.z, o4.w};
  const unsigned ps[4] = {p4.x, p4.y, p4.z, p4.w};
  const unsigned long long lt = L[t];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (o[s] < 0) continue;
    const unsigned long long lo = L[o[s]];
    if ((lo >> 1) != (lt >> 1) || ((lo ^ lt ^ ps[s] ^ 1u) & 1ull)) atomicOr(bad, 1);
  }
}

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 dsub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double ddot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 dcross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Element fields in host_setup.cpp's operation order (compiled -fmad=false).
__global__ void k_fields(long long K, const int4* cells, const double* coords, const int* other,
                         const unsigned long long* L, int* verts, int* neighbor, double* center,
                         double* radius, double* volume, double* diam, double* inv_edges,
                         unsigned long long* degenerate) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const bool flip = L[t] & 1ull;
  const int4 c = cells[t];
  int w[4] = {c.x, c.y, c.z, c.w};
  if (flip) {
    const int x = w[2];
    w[2] = w[3];
    w[3] = x;
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    verts[4 * t + s] = w[s];
    const int eff = flip ? (s == 2 ? 3 : (s == 3 ? 2 : s)) : s;
    neighbor[4 * t + eff] = other[4 * t + s];
  }
  D3 v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = {coords[3 * (long long)w[i]], coords[3 * (long long)w[i] + 1],
            coords[3 * (long long)w[i] + 2]};
  D3 cs = v[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) cs = {cs.x + v[i].x, cs.y + v[i].y, cs.z + v[i].z};
  const double q = 1.0 / 4;
  const D3 cen = {q * cs.x, q * cs.y, q * cs.z};
  double r2 = 0, d2 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const D3 dc = dsub(v[i], cen);
    r2 = fmax(r2, ddot(dc, dc));
#pragma unroll
    for (int j = i + 1; j < 4; ++j) {
      const D3 e = dsub(v[i], v[j]);
      d2 = fmax(d2, ddot(e, e));
    }
  }
  center[3 * t] = cen.x;
  center[3 * t + 1] = cen.y;
  center[3 * t + 2] = cen.z;
  radius[t] = sqrt(r2);
  diam[t] = sqrt(d2);
  const D3 e1 = dsub(v[1], v[0]), e2 = dsub(v[2], v[0]), e3 = dsub(v[3], v[0]);
  volume[t] = fabs(ddot(dcross(e1, e2), e3)) / 6.0;
  const double det = ddot(e1, dcross(e2, e3));
  if (det == 0) atomicMin(degenerate, (unsigned long long)t);
  const D3 r1 = dcross(e2, e3), rr2 = dcross(e3, e1), r3 = dcross(e1, e2);
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

__global__ void k_constrain(long long K, const int4* cells, const unsigned char* region,
                            unsigned char* constrained) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K || !region[t]) return;
  const int4 c = cells[t];
  constrained[c.x] = 1;
  constrained[c.y] = 1;
  constrained[c.z] = 1;
  constrained[c.w] = 1;
}

__global__ void k_free_flags(long long V, const unsigned char* constrained, int* flag) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V) flag[v] = constrained[v] ? 0 : 1;
}

__global__ void k_dof_ids(long long V, const unsigned char* constrained, int* dof) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < V && constrained[v]) dof[v] = -1;
}

template <class T>
void exclusive_scan(const T* in, T* out, long long n, cudaStream_t st) {
  size_t bytes = 0;
  CKS(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
  DBuf<unsigned char> tmp;
  tmp.alloc((long long)bytes);
  CKS(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, st));
}

template <class T>
T read1(const T* p) {
  T h;
  CKS(cudaMemcpy(&h, p, sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

}  // namespace

extern "C" int nlfem_gpu_element_table(const double* coords, int64_t nnodes, const int32_t* cells,
                                       const uint8_t* region, int64_t ncells, int32_t* verts,
                                       int32_t* neighbor, double* center, double* radius,
                                       double* volume, double* diam, double* inv_edges,
                                       int32_t* dof_of_node, uint8_t* constrained,
                                       int32_t* unknowns, int32_t device, char* err,
                                       size_t errlen) {
  auto say = [&](const std::string& m) {
    if (err && errlen) std::snprintf(err, errlen, "%s", m.c_str());
  };
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    say("no CUDA device available (the GPU setup has no CPU fallback)");
    return NLFEM_GPU_ENODEVICE;
  }
  try {
    if (device >= 0) CKS(cudaSetDevice(device));
    const long long K = ncells, V = nnodes;
    const cudaStream_t st = 0;
    DBuf<double> dco;
    DBuf<int4> dce;
    DBuf<unsigned char> dreg;
    dco.alloc(3 * V);
    dce.alloc(K);
    dreg.alloc(K);
    if (V) CKS(cudaMemcpy(dco.p, coords, sizeof(double) * 3 * V, cudaMemcpyHostToDevice));
    if (K) {
      CKS(cudaMemcpy(dce.p, cells, sizeof(int4) * K, cudaMemcpyHostToDevice));
      CKS(cudaMemcpy(dreg.p, region, K, cudaMemcpyHostToDevice));
    }
    // --- validation
    DBuf<unsigned> deg;
    DBuf<unsigned long long> flags;  // [0] bad key, [1] dangling, [2] degenerate
    DBuf<int> iflags;                // [0] nonmanifold, [1] changed, [2] not orientable
    deg.alloc(V);
    flags.alloc(3);
    iflags.alloc(3);
    CKS(cudaMemsetAsync(deg.p, 0, sizeof(unsigned) * std::max(V, 1LL), st));
    CKS(cudaMemsetAsync(flags.p, 0xff, sizeof(unsigned long long) * 3, st));
    CKS(cudaMemsetAsync(iflags.p, 0, sizeof(int) * 3, st));
    if (K) k_validate<<<blocks(K), kThr, 0, st>>>(dce.p, K, V, deg.p, flags.p);
    const unsigned long long badkey = read1(flags.p);
    if (badkey != ~0ull) {
      const long long k = (long long)(badkey >> 3);
      const int i = int(badkey >> 1 & 3);
      const int v = cells[4 * k + i];
      say("BadIndex: cell " + std::to_string(k) + (badkey & 1 ? " repeats vertex " : " references vertex ") +
          std::to_string(v));
      return NLFEM_GPU_BAD_INDEX;
    }
    if (V) k_dangling<<<blocks(V), kThr, 0, st>>>(deg.p, V, flags.p + 1);
    const unsigned long long dang = read1(flags.p + 1);
    if (dang != ~0ull) {
      say("DanglingVertex: vertex " + std::to_string(dang) + " is not used by any cell");
      return NLFEM_GPU_DANGLING_VERTEX;
    }
    // --- node -> cell incidence, facet gluing
    DBuf<long long> cnt, off;
    DBuf<int> inc;
    cnt.alloc(V + 1);
    off.alloc(V + 1);
    inc.alloc(4 * K);
    CKS(cudaMemsetAsync(cnt.p + V, 0, sizeof(long long), st));
    if (V) k_widen<<<blocks(V), kThr, 0, st>>>(deg.p, V, cnt.p);
    exclusive_scan(cnt.p, off.p, V + 1, st);
    CKS(cudaMemsetAsync(deg.p, 0, sizeof(unsigned) * std::max(V, 1LL), st));
    if (K) k_incidence<<<blocks(K), kThr, 0, st>>>(dce.p, K, off.p, deg.p, inc.p);
    DBuf<int> other;
    DBuf<unsigned char> psum;
    other.alloc(4 * K);
    psum.alloc(4 * K);
    if (K) k_match<<<blocks(4 * K), kThr, 0, st>>>(dce.p, K, off.p, inc.p, other.p, psum.p,
                                                    iflags.p);
    if (read1(iflags.p)) {
      say("NonManifold: facet shared by more than two cells");
      return NLFEM_GPU_NON_MANIFOLD;
    }
    // --- orientation labels
    DBuf<unsigned long long> L;
    L.alloc(K);
    if (K) k_label_init<<<blocks(K), kThr, 0, st>>>(K, L.p);
    for (long long it = 0; K && it <= K; ++it) {
      CKS(cudaMemsetAsync(iflags.p + 1, 0, sizeof(int), st));
      k_label_relax<<<blocks(K), kThr, 0, st>>>(K, reinterpret_cast<const int4*>(other.p),
                                                reinterpret_cast<const uchar4*>(psum.p), L.p,
                                                iflags.p + 1);
      if (!read1(iflags.p + 1)) break;
    }
    if (K)
      k_label_check<<<blocks(K), kThr, 0, st>>>(K, reinterpret_cast<const int4*>(other.p),
                                                reinterpret_cast<const uchar4*>(psum.p), L.p,
                                                iflags.p + 2);
    if (read1(iflags.p + 2)) {
      say("NonManifold: mesh is not orientable");
      return NLFEM_GPU_NON_MANIFOLD;
    }
    // --- element fields
    DBuf<int> dverts, dnb;
    DBuf<double> dcen, drad, dvol, ddia, dinv;
    dverts.alloc(4 * K);
    dnb.alloc(4 * K);
    dcen.alloc(3 * K);
    drad.alloc(K);
    dvol.alloc(K);
    ddia.alloc(K);
    dinv.alloc(9 * K);
    if (K)
      k_fields<<<blocks(K), kThr, 0, st>>>(K, dce.p, dco.p, other.p, L.p, dverts.p, dnb.p,
                                           dcen.p, drad.p, dvol.p, ddia.p, dinv.p, flags.p + 2);
    const unsigned long long degen = read1(flags.p + 2);
    if (degen != ~0ull) {
      say("BadConfig: degenerate element " + std::to_string(degen));
      return NLFEM_GPU_BAD_CONFIG;
    }
    // --- dof map
    DBuf<unsigned char> dcon;
    DBuf<int> dfree, ddof;
    dcon.alloc(V);
    dfree.alloc(V + 1);
    ddof.alloc(V + 1);
    CKS(cudaMemsetAsync(dcon.p, 0, std::max(V, 1LL), st));
    CKS(cudaMemsetAsync(dfree.p + V, 0, sizeof(int), st));
    if (K) k_constrain<<<blocks(K), kThr, 0, st>>>(K, dce.p, dreg.p, dcon.p);
    if (V) k_free_flags<<<blocks(V), kThr, 0, st>>>(V, dcon.p, dfree.p);
    exclusive_scan(dfree.p, ddof.p, V + 1, st);
    if (V) k_dof_ids<<<blocks(V), kThr, 0, st>>>(V, dcon.p, ddof.p);
    CKS(cudaGetLastError());
    // --- results to the host
    auto down = [&](void* h, const void* d, size_t bytes) {
      if (bytes) CKS(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost));
    };
    down(verts, dverts.p, sizeof(int) * 4 * K);
    down(neighbor, dnb.p, sizeof(int) * 4 * K);
    down(center, dcen.p, sizeof(double) * 3 * K);
    down(radius, drad.p, sizeof(double) * K);
    down(volume, dvol.p, sizeof(double) * K);
    down(diam, ddia.p, sizeof(double) * K);
    down(inv_edges, dinv.p, sizeof(double) * 9 * K);
    down(dof_of_node, ddof.p, sizeof(int) * V);
    down(constrained, dcon.p, V);
    *unknowns = read1(ddof.p + V);
    return 0;
  } catch (const SetupFail& f) {
    say(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    say(e.what());
    return NLFEM_GPU_ENODEVICE;
  }
}
