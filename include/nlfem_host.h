/* nlfem_host.h -- host-side setup that feeds nlfem_gpu_assemble().
 *
 * The reference keeps mesh generation, the combinatorial map, the element
 * table, the dof map and the manufactured problem on the host; so do we.
 * These are C restatements of that upstream (not timed by the assembly
 * metric, not GPU code), so the GPU box can build the same inputs without the
 * reference.  Each produces bit-identical arrays to the reference function it
 * cites (pinned by tests/test_host_setup.py against oracle/_ref).
 */
#ifndef NLFEM_HOST_H
#define NLFEM_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Structured 3D mesh of generate_mesh(3, res, delta) (reference mesh.cpp:115-121,
 * lattice 24-90): cube indices [-L, res+L)^3, L = ceil(delta*res - 1e-9), six
 * Kuhn tets per cube, region 1 outside [0,1]^3.
 * jitter_seed >= 0 additionally moves every node with lattice indices strictly
 * inside (0,res)^3 by h*(0.4*u - 0.2) per axis, u from xoshiro256++ seeded like
 * nlfem::Rng(jitter_seed) (reference core.hpp:108-133), three draws per node in
 * node-id order (the builder-defined config-3 recipe).
 * Call with NULL outputs to get the sizes. */
int nlfem_host_lattice_mesh(int32_t res, double delta, int64_t jitter_seed,
                            int64_t* nnodes, int64_t* ncells, double* coords,
                            int32_t* cells, uint8_t* region);

/* build_cmap + build_element_table (reference cmap.cpp:56-278,
 * ball_approx.cpp:33-98) for a 3D mesh: validates indices, orients cells
 * consistently (the last two vertices of a flipped cell swap), and fills every
 * ElementTable field.  Returns nlfem_gpu_status codes (BAD_INDEX,
 * DANGLING_VERTEX, NON_MANIFOLD, BAD_CONFIG for a degenerate element). */
int nlfem_host_element_table(const double* coords, int64_t nnodes, const int32_t* cells,
                             const uint8_t* region, int64_t ncells, int32_t* verts,
                             int32_t* neighbor, double* center, double* radius,
                             double* volume, double* diam, double* inv_edges, char* err,
                             size_t errlen);

/* build_dofmap (reference assembly.cpp:16-40).  Returns the unknown count. */
int32_t nlfem_host_dofmap(const int32_t* verts, const uint8_t* region, int64_t ncells,
                          int64_t nnodes, int32_t* dof_of_node, uint8_t* constrained);

/* make_kernel(3, delta, norm).C (reference polynomial.cpp:112-125);
 * moment2 != 0 selects Normalization::SecondMoment. */
double nlfem_host_kernel_constant(double delta, int32_t moment2);

/* f = -L u for polynomial u (reference problem.cpp:5-11, polynomial.cpp:127-150).
 * Terms are (c, e0, e1, e2) rows; returns the number of f terms written. */
int32_t nlfem_host_forcing(double delta, int32_t moment2, const double* uterms,
                           int32_t nu, double* fterms, int32_t maxterms);

/* Normalised polynomial (sorted, merged, zero-free), as Polynomial stores it. */
int32_t nlfem_host_normalize_poly(const double* terms, int32_t n, double* out,
                                  int32_t maxterms);

#ifdef __cplusplus
}
#endif
#endif /* NLFEM_HOST_H */
