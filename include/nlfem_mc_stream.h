/* nlfem_mc_stream.h -- definition of the counter-based Monte Carlo sample
 * stream for fullcaps ("mode P").  Host and device compile the same code, so
 * the GPU kernels and the CPU oracle draw the same points and take the same
 * accept decisions bit for bit.
 *
 * What stays the reference's (assembly.cpp:383-399, ball_approx.cpp:257-298):
 *   - the Monte Carlo regions: straddle_outer sub-simplices of a straddling
 *     element, or the whole element when all vertices are outside but it meets
 *     the ball;
 *   - mc_samples draws per sub-simplex, weight vol(sub)/mc_samples per hit,
 *     accept iff |y - x_q|^2 < delta^2;
 *   - uniform points by sorted spacings (quadrature.cpp:94-108).
 * What is ours (the reference uses xoshiro256++ keyed by a walk-order piece
 * index, assembly.cpp:386-387, which a parallel kernel cannot reproduce):
 *   - Philox4x32-10 (Salmon et al. 2011; Random123 constants), key =
 *     (seed & 0xffffffff, seed >> 32);
 *   - sample k of sub-simplex `sub` of item (outer elem T, quad pt q, inner
 *     elem T') uses block j = k / 4 of counters
 *         (T, T', q | sub << 2, 3j + c),  c = 0, 1, 2
 *     whose 12 output words W[0..11] give uniforms W[3i], W[3i+1], W[3i+2] to
 *     sample k = 4j + i;
 *   - u = (w + 0.5) * 2^-32, the three sorted as integers first;
 *   - the point relative to x_q, with sorted u0 <= u1 <= u2 and sub-simplex
 *     vertices V0..V3:  r = (V3 - x_q) + u0 (V0-V1) + u1 (V1-V2) + u2 (V2-V3),
 *     evaluated with the fused multiply-adds written below (this is the
 *     reference's  y = u0 V0 + (u1-u0) V1 + (u2-u1) V2 + (1-u2) V3  regrouped);
 *   - accept iff fma(rz, rz, fma(ry, ry, rx*rx)) < delta*delta.
 */
#ifndef NLFEM_MC_STREAM_H
#define NLFEM_MC_STREAM_H

#include <stdint.h>

#if defined(__CUDACC__)
#define NLFEM_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define NLFEM_HD static inline
#endif

#define NLFEM_PHILOX_M0 0xD2511F53u
#define NLFEM_PHILOX_M1 0xCD9E8D57u
#define NLFEM_PHILOX_W0 0x9E3779B9u
#define NLFEM_PHILOX_W1 0xBB67AE85u

NLFEM_HD void nlfem_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
#if defined(__CUDA_ARCH__)
  *hi = __umulhi(a, b);
  *lo = a * b;
#else
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
#endif
}

/* Philox4x32 with 10 rounds. */
NLFEM_HD void nlfem_philox4x32_10(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1,
                                  uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    nlfem_mulhilo32(NLFEM_PHILOX_M0, c0, &hi0, &lo0);
    nlfem_mulhilo32(NLFEM_PHILOX_M1, c2, &hi1, &lo1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += NLFEM_PHILOX_W0;
    k1 += NLFEM_PHILOX_W1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* The 12 words of sample block j of sub-simplex `sub` of item (T, q, T'). */
NLFEM_HD void nlfem_mc_block(uint64_t seed, uint32_t T, uint32_t Tp, uint32_t q,
                             uint32_t sub, uint32_t j, uint32_t W[12]) {
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (uint32_t c = 0; c < 3; ++c) {
    const uint32_t ctr[4] = {T, Tp, q | (sub << 2), 3u * j + c};
    nlfem_philox4x32_10(ctr, k0, k1, W + 4 * c);
  }
}

NLFEM_HD double nlfem_u01(uint32_t w) { return ((double)w + 0.5) * 0x1.0p-32; }

NLFEM_HD void nlfem_sort3u(uint32_t* a, uint32_t* b, uint32_t* c) {
  uint32_t x = *a, y = *b, z = *c, t;
  if (x > y) { t = x; x = y; y = t; }
  if (y > z) { t = y; y = z; z = t; }
  if (x > y) { t = x; x = y; y = t; }
  *a = x;
  *b = y;
  *c = z;
}

/* Sub-simplex frame for sampling: E0 = V0-V1, E1 = V1-V2, E2 = V2-V3,
 * P = V3 - x_q (plain IEEE subtractions). */
typedef struct {
  double e0[3], e1[3], e2[3], p[3];
} nlfem_mc_frame;

NLFEM_HD void nlfem_mc_make_frame(const double v0[3], const double v1[3], const double v2[3],
                                  const double v3[3], const double xq[3], nlfem_mc_frame* f) {
  for (int a = 0; a < 3; ++a) {
    f->e0[a] = v0[a] - v1[a];
    f->e1[a] = v1[a] - v2[a];
    f->e2[a] = v2[a] - v3[a];
    f->p[a] = v3[a] - xq[a];
  }
}

/* One sample from three raw words: writes r = y - x_q, returns 1 on a hit. */
NLFEM_HD int nlfem_mc_point(uint32_t w0, uint32_t w1, uint32_t w2, const nlfem_mc_frame* f,
                            double dd, double r[3]) {
  nlfem_sort3u(&w0, &w1, &w2);
  const double u0 = nlfem_u01(w0), u1 = nlfem_u01(w1), u2 = nlfem_u01(w2);
  for (int a = 0; a < 3; ++a)
    r[a] = fma(u2, f->e2[a], fma(u1, f->e1[a], fma(u0, f->e0[a], f->p[a])));
  const double d2 = fma(r[2], r[2], fma(r[1], r[1], r[0] * r[0]));
  return d2 < dd;
}

#endif /* NLFEM_MC_STREAM_H */
