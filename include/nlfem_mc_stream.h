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
 *   - uniform points by sorted spacings (quadrature.cpp:94-108):
 *     y = u0 V0 + (u1-u0) V1 + (u2-u1) V2 + (1-u2) V3, u0 <= u1 <= u2.
 * What is ours (the reference uses xoshiro256++ keyed by a walk-order piece
 * index, assembly.cpp:386-387, which a parallel kernel cannot reproduce):
 *   - Philox4x32 (Salmon et al. 2011; Random123 constants) with
 *     NLFEM_MC_ROUNDS = 7 rounds, key = (seed & 0xffffffff, seed >> 32).
 *     Seven is the round count Salmon et al. found to be the smallest that
 *     passes TestU01's BigCrush for every counter/key pattern they tried
 *     ("Crush-resistant"); ten is Random123's default, which adds a safety
 *     margin.  The 3D stream takes seven (round 2: 9% off the Monte Carlo
 *     kernel, whose integer issue is a third Philox); the 2D stream below and
 *     the known-answer tests use ten;
 *   - samples come in blocks of four: block j of sub-simplex `sub` of item
 *     (outer elem T, quad pt q, inner elem T') is the 8 words W[0..7] of the
 *     counters  (T, T', q | sub << 2, 2j + c),  c = 0, 1;  sample k = 4j + i;
 *   - each sample takes three 21-bit fields (two samples per Philox output):
 *     sample 2c   : W[4c] >> 11, W[4c+1] >> 11, W[4c+2] >> 11
 *     sample 2c+1 : ((W[4c+t] & 0x7ff) << 10) | ((W[4c+3] >> (22 - 10 t)) & 0x3ff),
 *                   t = 0, 1, 2;
 *     sorted s0 <= s1 <= s2 as integers, u_t = (s_t + 1/2) 2^-21;
 *   - with F_t = 2^-21 E_t (E0 = V0-V1, E1 = V1-V2, E2 = V2-V3, exact power-of-
 *     two scaling) the point is y - x_q = a + s0 F0 + s1 F1 + s2 F2,
 *     a = (V3 - x_q) + (F0 + F1 + F2)/2 (the spacings formula regrouped), and
 *     the hit test evaluates |y - x_q|^2 as the quadratic form in s,
 *         Q(s) = c + s.(b + A s),   c = |a|^2, b_t = 2 F_t.a, A_tu = F_t.F_u,
 *     in the fused multiply-add order written below: accept iff Q < delta^2.
 *     (No point is formed for the test; the GPU accumulates the exact integer
 *     moments sum s, sum s s^T of the hits and maps them through a and F once
 *     per sub-simplex.)
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

/* Rounds of the 3D Monte Carlo stream (see the header comment). */
#define NLFEM_MC_ROUNDS 7

/* Philox4x32 with `rounds` rounds (Philox4x32-R: the same round function R
 * times; the first rounds of Philox4x32-10 are Philox4x32-7). */
NLFEM_HD void nlfem_philox4x32_r(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1,
                                 int rounds, uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < rounds; ++r) {
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

/* Philox4x32-10 (Random123's default; the 2D stream and the KATs). */
NLFEM_HD void nlfem_philox4x32_10(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1,
                                  uint32_t out[4]) {
  nlfem_philox4x32_r(ctr_in, k0, k1, 10, out);
}

/* The 8 words of sample block j of sub-simplex `sub` of item (T, q, T'). */
NLFEM_HD void nlfem_mc_block(uint64_t seed, uint32_t T, uint32_t Tp, uint32_t q,
                             uint32_t sub, uint32_t j, uint32_t W[8]) {
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (uint32_t c = 0; c < 2; ++c) {
    const uint32_t ctr[4] = {T, Tp, q | (sub << 2), 2u * j + c};
    nlfem_philox4x32_r(ctr, k0, k1, NLFEM_MC_ROUNDS, W + 4 * c);
  }
}

/* The three 21-bit fields of sample i (0..3) of a block. */
NLFEM_HD void nlfem_mc_fields(const uint32_t W[8], int i, uint32_t f[3]) {
  const uint32_t* w = W + 4 * (i >> 1);
  if ((i & 1) == 0) {
    f[0] = w[0] >> 11;
    f[1] = w[1] >> 11;
    f[2] = w[2] >> 11;
  } else {
    f[0] = ((w[0] & 0x7ffu) << 10) | ((w[3] >> 22) & 0x3ffu);
    f[1] = ((w[1] & 0x7ffu) << 10) | ((w[3] >> 12) & 0x3ffu);
    f[2] = ((w[2] & 0x7ffu) << 10) | ((w[3] >> 2) & 0x3ffu);
  }
}

NLFEM_HD void nlfem_sort3u(uint32_t* a, uint32_t* b, uint32_t* c) {
  uint32_t x = *a, y = *b, z = *c, t;
  if (x > y) { t = x; x = y; y = t; }
  if (y > z) { t = y; y = z; z = t; }
  if (x > y) { t = x; x = y; y = t; }
  *a = x;
  *b = y;
  *c = z;
}

/* Per-sub-simplex constants: F_t = 2^-21 E_t (rows), a, and the quadratic
 * form Q(s) = c + s.(b + A s) of |y - x_q|^2 (A2 = off-diagonals doubled). */
typedef struct {
  double F[3][3], a[3];
  double c, b[3], A[3], A2[3]; /* A: 00 11 22; A2: 2*01 2*02 2*12 */
} nlfem_mc_quad;

NLFEM_HD double nlfem_dot3(const double x[3], const double y[3]) {
  return fma(x[2], y[2], fma(x[1], y[1], x[0] * y[0]));
}

NLFEM_HD void nlfem_mc_make_quad(const double v0[3], const double v1[3], const double v2[3],
                                 const double v3[3], const double xq[3], nlfem_mc_quad* Q) {
  for (int t = 0; t < 3; ++t) {
    Q->F[0][t] = (v0[t] - v1[t]) * 0x1p-21;
    Q->F[1][t] = (v1[t] - v2[t]) * 0x1p-21;
    Q->F[2][t] = (v2[t] - v3[t]) * 0x1p-21;
  }
  for (int t = 0; t < 3; ++t)
    Q->a[t] = (v3[t] - xq[t]) + ((Q->F[0][t] + Q->F[1][t]) + Q->F[2][t]) * 0.5;
  Q->c = nlfem_dot3(Q->a, Q->a);
  for (int t = 0; t < 3; ++t) {
    Q->b[t] = 2.0 * nlfem_dot3(Q->F[t], Q->a);
    Q->A[t] = nlfem_dot3(Q->F[t], Q->F[t]);
  }
  Q->A2[0] = 2.0 * nlfem_dot3(Q->F[0], Q->F[1]);
  Q->A2[1] = 2.0 * nlfem_dot3(Q->F[0], Q->F[2]);
  Q->A2[2] = 2.0 * nlfem_dot3(Q->F[1], Q->F[2]);
}

/* Q(s) for the sorted fields as exact doubles d_t = s_t. */
NLFEM_HD double nlfem_mc_q(const nlfem_mc_quad* Q, double d0, double d1, double d2) {
  const double t0 = fma(Q->A[0], d0, fma(Q->A2[0], d1, fma(Q->A2[1], d2, Q->b[0])));
  const double t1 = fma(Q->A[1], d1, fma(Q->A2[2], d2, Q->b[1]));
  const double t2 = fma(Q->A[2], d2, Q->b[2]);
  return fma(d0, t0, fma(d1, t1, fma(d2, t2, Q->c)));
}

/* The sample's offset r = y - x_q = a + F^T d (for per-hit evaluations). */
NLFEM_HD void nlfem_mc_r(const nlfem_mc_quad* Q, double d0, double d1, double d2, double r[3]) {
  for (int t = 0; t < 3; ++t)
    r[t] = fma(d2, Q->F[2][t], fma(d1, Q->F[1][t], fma(d0, Q->F[0][t], Q->a[t])));
}

/* One sample i of a block: the sorted fields as doubles; returns 1 on a hit. */
NLFEM_HD int nlfem_mc_sample(const uint32_t W[8], int i, const nlfem_mc_quad* Q, double dd,
                             double d[3]) {
  uint32_t f[3];
  nlfem_mc_fields(W, i, f);
  nlfem_sort3u(&f[0], &f[1], &f[2]);
  d[0] = (double)f[0];
  d[1] = (double)f[1];
  d[2] = (double)f[2];
  return nlfem_mc_q(Q, d[0], d[1], d[2]) < dd;
}

/* ---- the two-dimensional stream (triangles, the reference's n == 2 path) ----
 * Sample k (0 <= k < M) of Monte Carlo sub-triangle `sub` of item (T, q, T'):
 * W = Philox4x32-10 of the counter (T, T', q | sub << 2, k >> 1), key as above;
 * its two uniforms are u_t = (W[2c + t] + 1/2) 2^-32, c = k & 1, t = 0, 1;
 * sorted u0 <= u1 (reference sample_simplex, quadrature.cpp:98-102) the point
 * is y = u0 V0 + (u1 - u0) V1 + (1 - u1) V2, summed left to right. */
NLFEM_HD void nlfem_mc2_block(uint32_t k0, uint32_t k1, uint32_t T, uint32_t Tp, uint32_t q,
                              uint32_t sub, uint32_t j, uint32_t W[4]) {
  const uint32_t ctr[4] = {T, Tp, q | (sub << 2), j};
  nlfem_philox4x32_10(ctr, k0, k1, W);
}

NLFEM_HD void nlfem_mc2_sample(const uint32_t W[4], int c, const double v0[3],
                               const double v1[3], const double v2[3], double y[3]) {
  double u0 = ((double)W[2 * c] + 0.5) * 0x1p-32, u1 = ((double)W[2 * c + 1] + 0.5) * 0x1p-32;
  if (u0 > u1) {
    const double t = u0;
    u0 = u1;
    u1 = t;
  }
  const double l0 = u0, l1 = u1 - u0, l2 = 1.0 - u1;
  for (int a = 0; a < 3; ++a) y[a] = (l0 * v0[a] + l1 * v1[a]) + l2 * v2[a];
}

#endif /* NLFEM_MC_STREAM_H */
