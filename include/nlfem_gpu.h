/* nlfem_gpu.h -- C-ABI of the B200 nonlocal stiffness assembler.
 *
 * Drop-in for the reference's hot path
 *
 *   LinearSystem nlfem::assemble(const ElementTable& et, const DofMap& dofs,
 *                                const Kernel& kernel, const ScalarFn& f,
 *                                const ScalarFn& g, const AssemblyConfig& cfg,
 *                                AssemblyStats* stats);
 *     (reference proj/include/nlfem/assembly.hpp:71-73, proj/src/assembly.cpp:617-843)
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Inputs are borrowed for the duration of a call.  Output arrays are owned by
 * the library and released with nlfem_gpu_free_csr() (whole-system downloads
 * live in one page-locked block from a process-wide pool, so the download is a
 * straight DMA; freeing returns the block to the pool).  Every entry point
 * returns 0 on success or an nlfem_gpu_status code, with a message in `err`.
 * There is no CPU fallback: without a usable sm_100 device the calls fail
 * with NLFEM_GPU_ENODEVICE.
 */
#ifndef NLFEM_GPU_H
#define NLFEM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  1..8 mirror nlfem::ErrorCode (reference core.hpp:18-27) in
 * declaration order + 1, so callers can rethrow nlfem::Error(code - 1, msg). */
enum nlfem_gpu_status {
  NLFEM_GPU_OK = 0,
  NLFEM_GPU_BAD_INDEX = 1,
  NLFEM_GPU_DANGLING_VERTEX = 2,
  NLFEM_GPU_NON_MANIFOLD = 3,
  NLFEM_GPU_SEED_MISMATCH = 4,
  NLFEM_GPU_BALL_EXITS_MESH = 5, /* reference assembly.cpp:710-719 */
  NLFEM_GPU_DEGENERATE_HULL = 6,
  NLFEM_GPU_BAD_MESH_FILE = 7,
  NLFEM_GPU_BAD_CONFIG = 8,      /* reference assembly.cpp:620-622 */
  NLFEM_GPU_ENODEVICE = 100,     /* no sm_100 device / CUDA error */
  NLFEM_GPU_ENOMEM = 101,
  NLFEM_GPU_EUNSUPPORTED = 102   /* reserved: a configuration the GPU path does not support */
};

/* Strategy ids follow nlfem::Strategy (reference ball_approx.hpp:17-24). */
enum nlfem_gpu_strategy {
  NLFEM_STRATEGY_INSIDE = 0,
  NLFEM_STRATEGY_OVERLAP = 1,
  NLFEM_STRATEGY_BARYCENTER = 2,
  NLFEM_STRATEGY_NOCAPS = 3,
  NLFEM_STRATEGY_APPROXCAPS = 4,
  NLFEM_STRATEGY_FULLCAPS = 5
};

/* Monte Carlo sample stream for fullcaps.
 * PHILOX: Philox4x32-10, key = (seed lo32, seed hi32), counter =
 * (outer elem, inner elem, quad pt, block); sample s of an item uses uniforms
 * 3s..3s+2.  Regions and estimator are the reference's
 * (assembly.cpp:383-399, ball_approx.cpp:257-298). */
enum nlfem_gpu_sampler { NLFEM_SAMPLER_PHILOX = 0 };

/* ElementTable (reference ball_approx.hpp:38-58) as flat host arrays.
 * Simplex vertices are node_xyz[verts[4t+i]] (ball_approx.cpp:56). */
typedef struct {
  int32_t node_count;
  int32_t elem_count;
  const double* node_xyz;   /* [node_count*3]  ElementTable::node            */
  const int32_t* verts;     /* [elem_count*4]  ElementTable::verts           */
  const int32_t* neighbor;  /* [elem_count*4]  ElementTable::neighbor, -1    */
  const double* center;     /* [elem_count*3]  ElementTable::center          */
  const double* radius;     /* [elem_count]    ElementTable::radius          */
  const double* volume;     /* [elem_count]    ElementTable::volume          */
  const double* diam;       /* [elem_count]    ElementTable::diam            */
  const uint8_t* region;    /* [elem_count]    ElementTable::region (0/1)    */
  const double* inv_edges;  /* [elem_count*9]  ElementTable::inv_edges       */
} nlfem_gpu_mesh;

/* ElementTable of a TWO-dimensional mesh (reference ball_approx.hpp:38-58 with
 * n == 2: P1 triangles, ball_approx.cpp:51-80): node coordinates keep the
 * reference's Vec layout (x, y, 0); three vertices / neighbours per element;
 * inv_edges holds the four 2x2 entries the reference fills for n == 2. */
typedef struct {
  int32_t node_count;
  int32_t elem_count;
  const double* node_xyz;   /* [node_count*3]  (z = 0)                         */
  const int32_t* verts;     /* [elem_count*3]                                  */
  const int32_t* neighbor;  /* [elem_count*3]  -1 = unglued facet              */
  const double* center;     /* [elem_count*3]                                  */
  const double* radius;     /* [elem_count]                                    */
  const double* volume;     /* [elem_count]    triangle area                   */
  const double* diam;       /* [elem_count]                                    */
  const uint8_t* region;    /* [elem_count]                                    */
  const double* inv_edges;  /* [elem_count*4]                                  */
} nlfem_gpu_mesh2d;

/* DofMap (reference assembly.hpp:19-26): dof_of_node[v] = -1 when constrained. */
typedef struct {
  int32_t node_count;
  int32_t unknowns;
  const int32_t* dof_of_node;
} nlfem_gpu_dofs;

/* Kernel (reference polynomial.hpp:36-46): C * 1[|x-y| < delta], 3D only. */
typedef struct {
  double C;
  double delta;
} nlfem_gpu_kernel;

/* Polynomial f or g (reference polynomial.hpp:13-25): terms in Polynomial
 * sort order; evaluated exactly as Polynomial::eval (polynomial.cpp:28-37). */
typedef struct {
  int32_t nterms;
  const double* coef;   /* [nterms]   */
  const int32_t* exps;  /* [nterms*3] */
} nlfem_gpu_poly;

/* AssemblyConfig (reference assembly.hpp:50-55). */
typedef struct {
  int32_t strategy;     /* nlfem_gpu_strategy                                  */
  int32_t mc_samples;   /* per Monte Carlo sub-simplex, as the reference       */
  uint64_t seed;
  int32_t sampler;      /* nlfem_gpu_sampler                                   */
  int32_t device;       /* CUDA device ordinal (-1: current)                    */
} nlfem_gpu_config;

/* LinearSystem (reference assembly.hpp:36-42): CSR with sorted columns. */
typedef struct {
  int32_t rows;
  int64_t nnz;
  int32_t* row_ptr;     /* [rows+1] (library-owned) */
  int32_t* col_idx;     /* [nnz]                    */
  double* values;       /* [nnz]                    */
  double* rhs;          /* [rows]                   */
} nlfem_gpu_csr;

/* AssemblyStats (reference assembly.hpp:57-63) plus GPU counters. */
typedef struct {
  double seconds;          /* wall time of the whole call                     */
  int32_t threads;         /* 1 (one host thread drives the device)           */
  int32_t blocks;          /* ceil(interior/32), the reference's block count  */
  uint64_t mc_samples;     /* draws, per MC sub-simplex semantics             */
  uint64_t mc_hits;
  int64_t element_pairs;   /* (T,T') with a piece for some quad point of T     */
  int64_t items;           /* (T,q,T') with pieces                            */
  int64_t nnz_ext;         /* node-pattern size incl. constrained columns     */
  double device_ms;        /* device pipeline time (CUDA events)              */
  double phase_ms[8];      /* prep, pairs, pattern, integrate, finalize, ...  */
  uint64_t ledger_flops;   /* algorithmic FP64 FLOPs of the integration kernel,
                              SURVEY.md 8(d) ledger (whole 39/133, crossing 38,
                              straddle volume 24, Gauss sub-simplex 360/160, MC
                              sub-simplex setup 25, sample 35, hit +62/+12)   */
  uint64_t mc_subsimplices;
  int64_t shard_pairs;     /* element pairs integrated by this run (its shard)  */
  uint64_t ledger_flops_units; /* the part of ledger_flops done by the units
                              kernels (k_mc / k_approx: inner pieces and Monte
                              Carlo), whose phase time is phase_ms[5]        */
} nlfem_gpu_stats;

/* One-shot drop-in: host arrays in, host CSR out (upload + device pipeline +
 * download inside the call).  The analogue of nlfem::assemble. */
int nlfem_gpu_assemble(const nlfem_gpu_mesh* mesh, const nlfem_gpu_dofs* dofs,
                       const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                       const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                       nlfem_gpu_csr* out, nlfem_gpu_stats* stats, char* err,
                       size_t errlen);

void nlfem_gpu_free_csr(nlfem_gpu_csr* csr);

/* Conjugate gradients on the assembled system (reference cg_solve,
 * proj/include/nlfem/solver.hpp, proj/src/solver.cpp:26-66): unpreconditioned,
 * x0 = 0, stops at the first iteration with ||r|| <= tol ||b|| or when p.Ap
 * loses positivity, at most max_iter iterations.  Deterministic (fixed-order
 * reductions).  _device takes device arrays (row offsets int64, e.g. from
 * nlfem_gpu_session_outputs) and a device x; nlfem_gpu_cg host arrays. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double relative_residual;
} nlfem_gpu_solve_report;

int nlfem_gpu_cg(const nlfem_gpu_csr* sys, const double* b, double tol, int32_t max_iter,
                 int32_t device, double* x, nlfem_gpu_solve_report* report, char* err,
                 size_t errlen);
int nlfem_gpu_cg_device(int32_t rows, const int64_t* row_off, const int32_t* col_idx,
                        const double* values, const double* b, double tol, int32_t max_iter,
                        double* x, void* stream, nlfem_gpu_solve_report* report, char* err,
                        size_t errlen);

/* The reference's upstream setup on the GPU: build_cmap (cmap.cpp:56-278),
 * build_element_table (ball_approx.cpp:51-95) and build_dofmap
 * (assembly.cpp:16-40) from raw (coords, cells, region) host arrays.  Writes
 * the same arrays as nlfem_host_element_table + nlfem_host_dofmap
 * (include/nlfem_host.h), bit for bit, and the same error codes and messages
 * (BAD_INDEX, DANGLING_VERTEX, NON_MANIFOLD, BAD_CONFIG for a degenerate
 * element).  device < 0: the current device. */
int nlfem_gpu_element_table(const double* coords, int64_t nnodes, const int32_t* cells,
                            const uint8_t* region, int64_t ncells, int32_t* verts,
                            int32_t* neighbor, double* center, double* radius, double* volume,
                            double* diam, double* inv_edges, int32_t* dof_of_node,
                            uint8_t* constrained, int32_t* unknowns, int32_t device, char* err,
                            size_t errlen);

/* Device-resident session: the mesh is uploaded once; run() executes the
 * device pipeline with inputs already in HBM and leaves the CSR on the device;
 * download() copies it out.  Not reentrant per session. */
typedef struct nlfem_gpu_session nlfem_gpu_session;

int nlfem_gpu_session_create(const nlfem_gpu_mesh* mesh, const nlfem_gpu_dofs* dofs,
                             const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                             const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                             nlfem_gpu_session** out, char* err, size_t errlen);
/* stream: a cudaStream_t (NULL = the legacy default stream). */
/* Reload a session with new inputs (same meaning as _create), reusing its
 * streams and device buffers: the workspace of repeated one-shot calls. */
int nlfem_gpu_session_reset(nlfem_gpu_session* s, const nlfem_gpu_mesh* mesh,
                            const nlfem_gpu_dofs* dofs, const nlfem_gpu_kernel* kernel,
                            const nlfem_gpu_poly* f, const nlfem_gpu_poly* g,
                            const nlfem_gpu_config* cfg, char* err, size_t errlen);
int nlfem_gpu_session_run(nlfem_gpu_session* s, void* stream, nlfem_gpu_stats* stats,
                          char* err, size_t errlen);
int nlfem_gpu_session_download(nlfem_gpu_session* s, nlfem_gpu_csr* out, char* err,
                               size_t errlen);
/* Multi-GPU building blocks (one process per GPU).
 * run_shard integrates only interior outer elements [lo, hi) (positions in
 * ascending interior-id order; pairs and node pattern are built for all), and
 * leaves the exact fixed-point partial sums on the device; finalize = 1 also
 * finalizes all rows (single-GPU use).  partials() exposes the device arrays
 * (V: int64 words, rhsT: doubles, each entry written by one shard only) for a
 * cross-rank integer sum (e.g. ncclAllReduce int64 / f64).  finalize() then
 * computes output rows [row_lo, row_hi) and download_rows() copies them out
 * (row_ptr relative to the block).  The summed result is bit-identical to a
 * single-GPU run for any sharding. */
int nlfem_gpu_session_run_shard(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                int32_t finalize, nlfem_gpu_stats* stats, char* err,
                                size_t errlen);
int nlfem_gpu_session_partials(nlfem_gpu_session* s, void** V, int64_t* nwords, void** rhsT,
                               int64_t* nrhs);
/* Sharded element pairs (multi-GPU without redundant pair construction).
 * pairs_shard builds the element pairs of outer elements [lo, hi) only (after
 * the mesh preprocessing) and returns their number; pairs_shard_out exposes
 * device views of the range's per-outer-element pair counts (int32, hi - lo)
 * and partner ids (int32, in outer order) for an all-gather; pairs_install takes
 * the gathered counts of ALL outer elements (int32, interior order) and all
 * partner ids (device pointers, concatenated in outer order) and makes the next
 * run_shard build the node pattern from them and integrate [lo, hi) with the
 * codes this rank computed.  Results are bit-identical to an unsharded run. */
int nlfem_gpu_session_pairs_shard(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                  int64_t* npairs, char* err, size_t errlen);
int nlfem_gpu_session_pairs_shard_out(nlfem_gpu_session* s, void** counts, void** partners,
                                      int64_t* npairs);
int nlfem_gpu_session_pairs_install(nlfem_gpu_session* s, void* stream, const void* counts,
                                    const void* partners, int64_t npairs_total, char* err,
                                    size_t errlen);
int nlfem_gpu_session_finalize(nlfem_gpu_session* s, void* stream, int32_t row_lo,
                               int32_t row_hi, char* err, size_t errlen);
/* Owner-computes multi-GPU (the north star's "each rank assembles its own row
 * block"; replaces the threads of the reference's worker pool,
 * assembly.cpp:746-776, by ranks).  Every rank:
 *   run_local(lo, hi)   builds the element pairs of outer elements [lo, hi)
 *                       only and a LOCAL node pattern (the rows those pairs
 *                       touch) and integrates them into it;
 *   halo_records(bounds) returns, grouped by destination rank (row block
 *                       r = unknowns [bounds[r], bounds[r+1])), one record per
 *                       local slot of an unknown row: key uint64 = node_row
 *                       << 32 | node_col, 4 int64 words (the slot's fixed-point
 *                       hi / lo and its mirror slot's hi / lo); counts[r] per
 *                       destination (device pointers, valid until the next
 *                       call);
 *   rhs_records(bounds) the load-vector partials (int32 interior position +
 *                       4 x 8 doubles) of the outer elements at each
 *                       destination's unknown nodes;
 *   finalize_merged     takes everything received for its row block
 *                       [row_lo, row_hi) (its own records included), sorts
 *                       the records, sums equal keys as integers and
 *                       finalizes the block; outputs() / download_rows() then
 *                       hold those rows.
 * Only the records move between ranks (an all-to-all of the halo); the
 * finalized row blocks are then all-gathered.  Bit-identical to one GPU. */
int nlfem_gpu_session_run_local(nlfem_gpu_session* s, void* stream, int32_t lo, int32_t hi,
                                nlfem_gpu_stats* stats, char* err, size_t errlen);
int nlfem_gpu_session_halo_records(nlfem_gpu_session* s, int32_t world, const int32_t* bounds,
                                   void** keys, void** vals, int64_t* counts, char* err,
                                   size_t errlen);
int nlfem_gpu_session_rhs_records(nlfem_gpu_session* s, int32_t world, const int32_t* bounds,
                                  void** idx, void** vals, int64_t* counts, char* err,
                                  size_t errlen);
int nlfem_gpu_session_finalize_merged(nlfem_gpu_session* s, void* stream, int32_t row_lo,
                                      int32_t row_hi, const void* keys, const void* vals,
                                      int64_t n, const void* ridx, const void* rvals, int64_t m,
                                      char* err, size_t errlen);
int nlfem_gpu_session_download_rows(nlfem_gpu_session* s, int32_t row_lo, int32_t row_hi,
                                    nlfem_gpu_csr* out, char* err, size_t errlen);
/* The reference's 2D path: nlfem::assemble with et.n == 2 (P1 triangles, disk
 * kernel; assembly.cpp:617-843) for all six strategies (approxcaps: the
 * reference's 2D sphere-point hull).  Same contract, errors
 * and outputs as nlfem_gpu_assemble; fullcaps draws from the two-dimensional
 * Philox stream of include/nlfem_mc_stream.h.  The entries are reduced by a
 * stable key sort and in-order sums (deterministic, no atomics on values). */
int nlfem_gpu_assemble_2d(const nlfem_gpu_mesh2d* mesh, const nlfem_gpu_dofs* dofs,
                          const nlfem_gpu_kernel* kernel, const nlfem_gpu_poly* f,
                          const nlfem_gpu_poly* g, const nlfem_gpu_config* cfg,
                          nlfem_gpu_csr* out, nlfem_gpu_stats* stats, char* err,
                          size_t errlen);

/* Device pointers of the output CSR of the last run (row offsets are int64,
 * columns int32, values and rhs double), for device-side collectives. */
int nlfem_gpu_session_outputs(nlfem_gpu_session* s, void** row_off, void** col_idx,
                              void** values, void** rhs, int32_t* rows, int64_t* nnz);

/* solve_problem + l2_error on the GPU (reference study.cpp:38-99): CG on the
 * session's assembled system where it lies in HBM (nlfem_gpu_cg_device, x0 = 0),
 * node values (unknowns from x, constrained nodes g(x_j), study.cpp:64-74),
 * the L2 error against `exact` with the 14-point degree-5 tetrahedral rule
 * over interior elements (study.cpp:76-99, quadrature.cpp:42-62) and the
 * largest nodal error max_j |u_h(x_j) - exact(x_j)|.  Deterministic
 * (fixed-order reductions).  u_node: optional host array [node_count]. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double relative_residual;
  double l2_error;
  double max_nodal_error;
  double device_ms; /* CG + node values + error norms, CUDA events */
} nlfem_gpu_study;

int nlfem_gpu_session_solve(nlfem_gpu_session* s, double tol, int32_t max_iter,
                            const nlfem_gpu_poly* exact, double* u_node, nlfem_gpu_study* out,
                            char* err, size_t errlen);


/* Element-pair list of the last run, for set parity: for each interior outer
 * element (in ascending id order) its partner ids and per-quad-point class
 * codes (5 bits per point) -- per (T, q) the parents the
 * reference's walk_ball emits pieces for (ball_approx.hpp:164-175).  Arrays sized by *npairs after a
 * call with NULL buffers. */
int nlfem_gpu_session_pairs(nlfem_gpu_session* s, int64_t* npairs, int64_t* outer_offsets,
                            int32_t* partner, uint32_t* info, char* err, size_t errlen);
/* The same element-pair list in place in device memory (valid until the
 * session's next run): outer offsets int64 [interior + 1], partner ids int32
 * and class codes uint32 [npairs]. */
int nlfem_gpu_session_pairs_device(nlfem_gpu_session* s, int64_t* npairs,
                                   const int64_t** outer_offsets, const int32_t** partner,
                                   const uint32_t** info);
/* Kernel launches of the last run (for the bench's gpu_launches key). */
int64_t nlfem_gpu_session_launches(const nlfem_gpu_session* s);
void nlfem_gpu_session_destroy(nlfem_gpu_session* s);

/* FP64 (non-tensor) DFMA throughput of the device, measured by a short
 * microbenchmark: the roofline denominator for the integration kernels
 * (MEASURED_PEAKS.json has no FP64 figure). */
int nlfem_gpu_fp64_peak(int32_t device, double* tflops, char* err, size_t errlen);

/* Checked builds (-DNLFEM_CHECKED=1) surround every device buffer with
 * canaries verified at the end of each run (an out-of-bounds write fails the
 * call).  This self-test writes one element past (past = 1) or at the end of
 * (past = 0) a fresh buffer: 1 = caught, 0 = not, -1 = default build, -2 = CUDA error. */
int nlfem_gpu_debug_guard_selftest(int32_t past);

/* Build / version string (e.g. "nlfem_gpu sm_100a ..."). */
const char* nlfem_gpu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NLFEM_GPU_H */
