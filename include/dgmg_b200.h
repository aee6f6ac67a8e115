/*
 * dgmg_b200.h - C ABI of the B200-native Schwarz-smoother hot path.
 *
 * Drop-in boundary for the reference package `dgmg` (arXiv 1910.11239,
 * /root/reference/pkg/src/dgmg).  The reference is pure Python; its hot path
 * is the fp64 Schwarz smoothing step on a uniform Cartesian SIPG level:
 *
 *   residual r = b - A x          dgop.residual        dgop.py:782-788
 *   operator v = A u              dgop.apply_operator  dgop.py:762-779
 *   cell FDM solves               CellSolverSet.solve_partitioned   fastdiag.py:457-496
 *   patch FDM solves              PatchSolverSet.solve_partitioned  fastdiag.py:602-628
 *   additive / multiplicative     LevelSmoother.smooth_additive / _multiplicative
 *                                 smoothers.py:131-166
 *
 * The Python mirror (paper_1910_11239_b200/) keeps those entry points and
 * binds the functions below through ctypes.
 *
 * Conventions
 *  - all vectors are device fp64 in the reference's canonical layout
 *    (cell-major, dof = cell*n^d + sum_t i_t n^(t-1), dgop.py:70-103);
 *  - every compute call is asynchronous on the caller's stream and returns
 *    DG_OK or an error code; dg_last_error() gives the thread-local message;
 *  - a level may hold a window of cell layers along the last direction
 *    (slab decomposition across GPUs): layers [z_begin, z_begin+z_count) of a
 *    global box with ncells[t] cells per direction are stored contiguously.
 */
#ifndef DGMG_B200_H
#define DGMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DG_OK = 0,
  DG_EINVAL = 1,      /* bad size / alias / argument  -> ValueError            */
  DG_ESINGULAR = 2,   /* nonpositive Kronecker eigenvalue sum (fastdiag.py:98) */
  DG_ECUDA = 3,       /* CUDA runtime failure                                  */
  DG_EUNSUPPORTED = 4 /* (dim, degree) without a compiled kernel               */
};

/* smoother kinds, SmootherConfig.kind (smoothers.py:41-69) */
enum { DG_ACS = 0, DG_MCS = 1, DG_AVS = 2, DG_MVS = 3 };

typedef struct dg_level_desc {
  int dim;            /* 2 or 3                                                */
  int degree;         /* k >= 1; n = k+1 nodes per direction                   */
  int ncells[3];      /* global cells per direction (unused entries = 1)       */
  int z_begin;        /* first stored layer along direction `dim`              */
  int z_count;        /* stored layers                                         */
  int own_begin;      /* owned layers [own_begin, own_end): cell solves/writes */
  int own_end;
  int res_begin;      /* layers whose residual dg_smooth computes              */
  int res_end;
  int pv_begin;       /* patch vertices v_dim in [pv_begin, pv_end] are solved */
  int pv_end;
} dg_level_desc_t;

/* Host tables from the 1D setup (paper_1910_11239_b200/tables.py).  All
 * matrices are row-major and applied as out_i = sum_k S[i*s+k] in_k.
 * `digit` (0..3) encodes the boundary pattern of one direction: bit 0 = left
 * face on the boundary, bit 1 = right face (fastdiag.py:349-369, 535-566).  */
typedef struct dg_tables {
  const double* mass;          /* n*n      1D cell mass M                      */
  const double* adiag;         /* 4*n*n    1D cell stiffness per digit         */
  const double* bg;            /* 2*n      basis derivatives at x=0, x=1       */
  double alpha;                /* -gamma_e/2  (rank-2 face coupling a_pm)      */
  double beta;                 /* -1/(2h)                                      */
  double betap;                /* +1/(2h)                                      */
  const double* cell_z;        /* 4*n*n    cell eigenvectors Z per digit       */
  const double* cell_zt;       /* 4*n*n    Z^T                                 */
  const double* cell_invsum;   /* 4^d*n^d  1/Lambda-sum per class, canonical   */
  const double* patch_z;       /* 4*m*m    patch eigenvectors, m = 2n (or NULL)*/
  const double* patch_zt;      /* 4*m*m                                        */
  const double* patch_invsum;  /* 4^d*m^d                                      */
  /* even/odd factorisation of the interior digit (NULL = dense everywhere):
   * the interior eigenpairs in cell_z/patch_z (and the class 1/Lambda tables)
   * must be ordered even-first; halves are (s/2)x(s/2), k-outer row-major:
   * *_eo = [Z_top_even, Z_top_odd, Z_top_even^T, Z_top_odd^T],
   * res_eo = [P^T, Q^T of M, P^T, Q^T of A_diag(0)] with
   * P = (A11 + A12 J)/2, Q = (A11 - A12 J)/2 (centro-symmetric splitting). */
  const double* cell_eo;       /* 4*(n/2)^2 or NULL                           */
  const double* patch_eo;      /* 4*(m/2)^2 or NULL                           */
  const double* res_eo;        /* 4*(n/2)^2 or NULL                           */
} dg_tables_t;

typedef struct dg_level dg_level_t;

const char* dg_last_error(void);
int dg_version(void);

/* Level lifetime: uploads the tables, builds the colour lists (red-black
 * cells, structured patch colours mesh.py:350-375) for the window.          */
int dg_level_create(const dg_level_desc_t* desc, const dg_tables_t* tables,
                    dg_level_t** out);
int dg_level_destroy(dg_level_t* lvl);

/* number of local dofs stored by the level (z_count layers)                 */
int64_t dg_level_ndofs(const dg_level_t* lvl);

/* v = A u on the cells of global layers [z0, z1) (dgop.apply_operator);
 * u, v are local vectors, v must not alias u.                               */
int dg_apply(const dg_level_t* lvl, const double* u, double* v,
             int z0, int z1, void* stream);
/* r = b - A x on the cells of layers [z0, z1) (dgop.residual)              */
int dg_residual(const dg_level_t* lvl, const double* x, const double* b,
                double* r, int z0, int z1, void* stream);
/* r = b - A x on an explicit list of local cell ids (device int32)         */
int dg_residual_cells(const dg_level_t* lvl, const double* x, const double* b,
                      double* r, const int32_t* cells, int64_t n_cells,
                      void* stream);

/* x[cell dofs] += omega * A_c^{-1} r_c for local cell ids (device int32), or
 * for all owned cells when cells == NULL (CellSolverSet.solve_partitioned). */
int dg_cell_fdm(const dg_level_t* lvl, const double* r, double* x,
                double omega, const int32_t* cells, int64_t n_cells,
                void* stream);
/* x[patch dofs] += omega * A_j^{-1} R_j r for global patch ids (device
 * int32).  atomic != 0 accumulates with fp64 atomics (overlapping patches,
 * safe_accumulate=True); otherwise the patches must be write-disjoint.     */
int dg_patch_fdm(const dg_level_t* lvl, const double* r, double* x,
                 double omega, const int32_t* patches, int64_t n_patches,
                 int atomic, void* stream);

/* Additive local solves restricted to a range of layers along the last
 * direction, for pipelined steps (host copies overlapped with compute):
 * DG_ACS: x += omega A_c^{-1} r_c for the owned cells with c_last in [lo, hi);
 * DG_AVS: x += omega R_j^T A_j^{-1} R_j r for the patches with last vertex
 * coordinate in [lo, hi), accumulated by fp64 bulk reduce-add (overlapping
 * patches may run concurrently).  (CellSolverSet / PatchSolverSet
 * .solve_partitioned, fastdiag.py:457-496, 602-628)                       */
int dg_solve_range(const dg_level_t* lvl, int kind, double omega, const double* r,
                   double* x, int lo, int hi, void* stream);

/* One colour of the multiplicative vertex-patch sweep restricted to the
 * patches whose last vertex coordinate is in [vlo, vhi) (colour = index of
 * the level's non-empty patch colours, sweep order): what & 1 computes the
 * restricted residual r = b - A x on their cells, what & 2 the local solves
 * x += omega A_j^-1 r_j (disjoint inside a colour).  The host wavefront
 * pipeline of LevelSmoother (smooth_multiplicative on host vectors) chains
 * these per z-chunk.  (LevelSmoother.smooth_multiplicative,
 * smoothers.py:157-166)                                                    */
int dg_mvs_range(const dg_level_t* lvl, int colour, int what, double omega, double* x,
                 const double* b, double* r, int vlo, int vhi, void* stream);

/* colour lists built at create time (device int32, owned by the level)     */
int dg_num_colours(const dg_level_t* lvl, int kind);
int dg_colour_list(const dg_level_t* lvl, int kind, int colour,
                   const int32_t** dev_ids, int64_t* count);
/* R_j gather map of patches [first, first+count) as local dof indices
 * (device int64, count*m^d), computed by the kernels' own index math.      */
int dg_patch_gather_map(const dg_level_t* lvl, const int32_t* patches,
                        int64_t count, int64_t* out, void* stream);

/* One smoothing step / sweep (LevelSmoother.smooth, smoothers.py:131-166):
 * ACS/AVS additive, MCS/MVS multiplicative (reverse flips colour order).
 * scratch_r holds the residual (local size).  The launch sequence is
 * captured once into a CUDA graph per (kind, omega, reverse, pointers) and
 * replayed when use_graph != 0.                                             */
int dg_smooth(dg_level_t* lvl, int kind, double omega, int reverse,
              double* x, const double* b, double* scratch_r, int use_graph,
              void* stream);

/* kernels launched by the last dg_smooth call (for the bench's count)      */
int64_t dg_last_launch_count(const dg_level_t* lvl);

/* 1 if the additive patch step (DG_AVS) of this level runs as the single
 * persistent dataflow kernel (residual + all colours, L2-resident z-blocks),
 * 0 if it runs as one residual launch plus one launch per colour.           */
int dg_flow_enabled(const dg_level_t* lvl);

/* Bit mask of optional code compiled into this library:
 * DG_BUILD_EXPERIMENTAL = the measured-and-rejected variants of DESIGN.md
 * section 8 (dataflow step DGB_FLOW, clusters DGB_CLUSTER, z-windowed and
 * overlapped AVS DGB_AVS_WIN / DGB_AVS_OVERLAP, persistent solves DGB_FDM=5/6,
 * DMMA solves DGB_MMA), built only with -DDGB_EXPERIMENTAL.                 */
#define DG_BUILD_EXPERIMENTAL 1
/* DG_BUILD_CHECKS = device-side bounds checks of every cell address
 * (-DDGB_CHECKS; a violation traps and the launch fails).                  */
#define DG_BUILD_CHECKS 2
int dg_build_flags(void);


/* Nested-level transfers between a coarse level with coarse_cells[t] cells
 * per direction and its uniform refinement (2*coarse_cells[t]); e0, e1 are
 * the host 1D embeddings E^s[i*n+j] = phi_j((x_i+s)/2) (build_transfer,
 * multigrid.py:51-55), n = degree+1.  Vectors are device fp64 canonical.
 * dg_prolongate: xf = P xc, or xf += P xc when accumulate != 0 (the
 *   V-cycle's coarse-grid correction, multigrid.py:340-341)
 *   (LevelTransfer.prolongate, multigrid.py:91-108);
 * dg_restrict:   xc = P^T xf (LevelTransfer.restrict, multigrid.py:110-130). */
int dg_prolongate(int dim, int degree, const int* coarse_cells, const double* e0,
                  const double* e1, const double* xc, double* xf, int accumulate,
                  void* stream);
int dg_restrict(int dim, int degree, const int* coarse_cells, const double* e0,
                const double* e1, const double* xf, double* xc, void* stream);

/* Setup-side tensor kernels (csrc/coarse.cu).  All pointers are device fp64.
 * dg_mode_contract: out[o,i,r] = sum_k S(i,k) in[o,k,r] for a tensor viewed as
 *   (outer, K, inner) -> (outer, I, inner); S is I x K row-major, or K x I
 *   row-major when transposed != 0.  One mode of a sum-factorised product:
 *   the load vector's basis contractions (`_tensor.backward_all`,
 *   _tensor.py:81-97, called by compute_rhs, dgop.py:800-871) and the passes
 *   of the coarse solve below.
 * dg_canonical_tensor: canonical cell-major vector (dgop.py:70-103) <->
 *   direction-major global tensor T[j_1 + N_1 (j_2 + N_2 j_3)], j_t = c_t n + i_t,
 *   N_t = ncells[t] n (to_tensor != 0: canonical -> tensor).
 * dg_kron_scale: T[j] /= lam0[j_1] + lam1[j_2] + lam2[j_3] (null = absent).
 * Together they apply A^-1 = (x)Z diag(1/sum lambda) (x)Z^T with the global
 * 1D eigenpairs of a Cartesian level: the exact coarse solve that stands in
 * for CoarseSolver's dense Cholesky / sparse LU (multigrid.py:169-195).      */
int dg_mode_contract(const double* in, double* out, const double* S, int64_t outer, int K,
                     int I, int64_t inner, int transposed, void* stream);
int dg_canonical_tensor(int dim, int degree, const int* ncells, const double* in, double* out,
                        int to_tensor, void* stream);
int dg_kron_scale(double* tensor, const double* lam0, const double* lam1, const double* lam2,
                  int n0, int n1, int n2, void* stream);

/* Fused vector kernels of the device-resident CG (krylov.pcg,
 * krylov.py:69-123).  `part` is device scratch of >= 1024 doubles, `out` one
 * device double receiving the (deterministic, fixed-order) reduction.
 * dg_cg_update: x += alpha p; r -= alpha ap; *out = r.r
 * dg_xpby:      p = z + beta p
 * dg_dot:       *out = a.b                                                 */
int dg_cg_update(double* x, double* r, const double* p, const double* ap, double alpha,
                 int64_t n, double* part, double* out, void* stream);
int dg_xpby(const double* z, double beta, double* p, int64_t n, void* stream);
int dg_dot(const double* a, const double* b, int64_t n, double* part, double* out,
           void* stream);

/* SIPG operator on a multilinear (distorted) cube level, SURVEY 8(f) row 3
 * (dgop.apply_operator / residual non-Cartesian branches, dgop.py:432-481,
 * 583-759).  Geometry arrays are device fp64 in the reference's layouts
 * (paper_1910_11239_b200/distorted.py builds them); tables are host arrays.
 * out = A u, or out = b - A u when b != NULL.                               */
typedef struct dg_dist_args {
  int dim, degree, ncells_dim;
  const double* metric;    /* (cells, n^d, d(d+1)/2) detJ J^-1 J^-T w        */
  const double* faces[3];  /* per direction: (faces, n^(d-1), 1 + 2d)        */
  const double* bnd[6];    /* per direction and side: (faces, n^(d-1), 1 + d) */
  const double* vals;      /* host (n, n): V[q][i] = phi_i(x_q)               */
  const double* grads;     /* host (n, n): D[q][i] = phi_i'(x_q)              */
  const double* bv;        /* host (2, n) basis values at x = 0, 1            */
  const double* bg;        /* host (2, n) basis derivatives at x = 0, 1       */
} dg_dist_args_t;
int dg_dist_apply(const dg_dist_args_t* args, const double* u, const double* b, double* out,
                  void* stream);
/* Surrogate cell solves on a multilinear level (CellSolverSet per-cell
 * batch, fastdiag.py:381-436, 457-496): x_c += omega Z Lambda_c^-1 Z^T r_c
 * with per-cell eigenbases z (dim, ncells, n, n) and 1/Lambda-sums inv
 * (ncells, n^dim, reversed layout), all device; cells NULL = every cell.    */
int dg_dist_cell_fdm(int dim, int degree, int64_t ncells, const double* z, const double* inv,
                     const double* r, double* x, double omega, const int32_t* cells,
                     int64_t n_cells, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DGMG_B200_H */
