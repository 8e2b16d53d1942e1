/*
 * mdd.h — C-ABI of libmdd.so, the B200-native (sm_100a) hot path behind the
 * reference package's Python API (maxwelldd, /root/reference/pkg/src/maxwelldd).
 *
 * The reference is pure Python; its "FFI" for this path is the set of Python
 * functions listed against each entry point below.  The Python host layer in
 * paper_1711_03789_b200/ binds these symbols with ctypes (paper_1711_03789_b200/
 * _lib.py) and keeps the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - complex128 is `mdd_complex` (two doubles, layout-identical to numpy
 *     complex128 and CUDA double2);
 *   - host pointers are caller-owned and only touched during the call;
 *   - device objects live behind opaque handles owned by the library;
 *   - every int-returning call returns an MDD_* code; on failure
 *     mdd_last_error() holds a thread-local message (reference exception text
 *     conventions: "subdomain {ell}: ...", "coarse space: ...").
 *   - there is no CPU fallback: a call needing a GPU fails with MDD_ECUDA when
 *     none is present.
 */
#ifndef MDD_H
#define MDD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } mdd_complex;

typedef struct mdd_ctx mdd_ctx;     /* one device + stream + scratch            */
typedef struct mdd_csr mdd_csr;     /* device CSR (int32 indptr/indices)        */
typedef struct mdd_space mdd_space; /* device mesh + edge space + CSR pattern   */
typedef struct mdd_prec mdd_prec;   /* factorised Schwarz preconditioner        */
typedef struct mdd_comm mdd_comm;   /* NCCL communicator (multi-GPU sharding)   */

enum {
  MDD_OK = 0,
  MDD_EINVAL = 1,    /* -> ValueError                                        */
  MDD_ESINGULAR = 2, /* -> linalg.SingularMatrixError (reference linalg.py:33) */
  MDD_ECAP = 3,      /* -> linalg.SizeCapError (reference linalg.py:37)        */
  MDD_ECUDA = 4,     /* CUDA runtime failure / no device                        */
  MDD_ENCCL = 5,
  MDD_ENOMEM = 6,
  MDD_EDECOMP = 7    /* -> decomp.DecompositionError (reference decomp.py:41)  */
};

/* ------------------------------------------------------------------ misc */
const char* mdd_last_error(void);
int mdd_version(void);
int mdd_device_count(int* n);

/* ---------------------------------------------------------------- context */
int mdd_ctx_create(int device, mdd_ctx** out);
void mdd_ctx_destroy(mdd_ctx* ctx);
int mdd_ctx_synchronize(mdd_ctx* ctx);
/* number of this library's kernels launched on the context so far */
int64_t mdd_ctx_kernel_launches(const mdd_ctx* ctx);
/* timers of the last mdd_gmres (ms): [0..2] device time of spmv / precond /
 * arnoldi (timing mode only), [3..5] host wall of setup / loop / finalisation,
 * [6] CUDA-graph construction */
int mdd_ctx_timers(const mdd_ctx* ctx, double* out8);
int mdd_ctx_set_timing(mdd_ctx* ctx, int enable);
/* CUDA events on the context stream (slot 0..15) for device-side timing */
int mdd_ctx_event_record(mdd_ctx* ctx, int slot);
int mdd_ctx_event_elapsed(mdd_ctx* ctx, int slot0, int slot1, double* ms);
/* device buffers (plumbing for device-resident benchmark inputs) */
int mdd_dev_alloc(mdd_ctx* ctx, int64_t bytes, void** out);
int mdd_dev_free(mdd_ctx* ctx, void* p);
int mdd_memcpy(mdd_ctx* ctx, void* dst, const void* src, int64_t bytes, int kind /*1 h2d, 2 d2h, 3 d2d*/);

/* ------------------------------------------------------------ CSR matrices
 * Replaces scipy.sparse CSR storage + linalg.spmv (reference linalg.py:41-45)
 * and the `a_mv = op @ v` of krylov._as_callable (reference krylov.py:58-61). */
int mdd_csr_from_host(mdd_ctx* ctx, int64_t nrow, int64_t ncol, int64_t nnz,
                      const int32_t* indptr, const int32_t* indices,
                      const void* values, int is_complex, mdd_csr** out);
int mdd_csr_info(const mdd_csr* A, int64_t* nrow, int64_t* ncol, int64_t* nnz,
                 int* is_complex);
int mdd_csr_to_host(const mdd_csr* A, int32_t* indptr, int32_t* indices, void* values);
void mdd_csr_destroy(mdd_csr* A);
/* y = A x with host vectors (complex; a real A acts on complex x) */
int mdd_spmv(mdd_ctx* ctx, const mdd_csr* A, const mdd_complex* x, mdd_complex* y);
/* timed device-resident SpMV loop for benchmarks: `reps` launches on device
 * buffers, returns the average kernel time (ms) measured with CUDA events.   */
int mdd_spmv_bench(mdd_ctx* ctx, const mdd_csr* A, int reps, double* ms_per_call);

/* ------------------------------------------------------- space + assembly
 * mdd_space_create uploads the mesh of reference mesh.build_cube_mesh
 * (mesh.py:126-213) and the DOF map of fem.build_edge_space (fem.py:71-80)
 * and builds the CSR pattern of fem._assemble_csr (fem.py:214-230). */
int mdd_space_create(mdd_ctx* ctx, int32_t cells_per_axis,
                     int64_t nv, const double* vertices,
                     int64_t nt, const int64_t* tets, const int64_t* tet_edges,
                     const int64_t* tet_edge_signs,
                     int64_t ne, const int64_t* edge_to_dof, int64_t ndof,
                     mdd_space** out);
void mdd_space_destroy(mdd_space* sp);
int mdd_space_nnz(const mdd_space* sp, int64_t* nnz);

/* Coefficients (reference fem.py:83-123). Arrays are per tet or NULL (then the
 * scalar eps0/mu0/sigma0 applies to all tets). */
typedef struct {
  double k, xi;
  const double* eps;
  const double* mu;
  const double* sigma;
  double eps0, mu0, sigma0;
  int homogeneous; /* Coefficients.homogeneous (fem.py:111-120) */
} mdd_coeffs;

/* fem.assemble (fem.py:233-279): A (complex), S, M, Dk (real) on the space's
 * pattern; impedance != 0 adds -i*sign(xi)*k*Mb over the nbf boundary faces
 * (sorted vertex triples) and returns Mb (fem.py:258-263, 319-353).  Any
 * output pointer may be NULL. */
int mdd_assemble(mdd_space* sp, const mdd_coeffs* co, int impedance,
                 int64_t nbf, const int64_t* bfaces,
                 mdd_csr** A, mdd_csr** S, mdd_csr** M, mdd_csr** Dk, mdd_csr** Mb);
/* Sharded solves (no reference counterpart: the reference assembles the whole matrix in one
 * process, fem.py:233-279): restrict the following mdd_assemble calls on this space to the
 * cells that touch an unknown in [row_lo, row_hi) -- the rows one rank needs (its subdomains'
 * unknowns and the columns of its owned rows, distributed.needed_rows).  Rows of the returned
 * matrices inside the window are complete and bitwise equal to the unrestricted assembly; rows
 * outside it are not.  row_lo < 0 (or the full range) removes the window. */
int mdd_space_set_row_window(mdd_space* sp, int64_t row_lo, int64_t row_hi);
/* fem.assemble_rhs (fem.py:373-390): fvals are the source values at the
 * 4-point rule's points, layout (4, nt, 3) complex; rhs is host (ndof). */
int mdd_assemble_rhs(mdd_space* sp, const mdd_complex* fvals, mdd_complex* rhs);
/* Same, with the source F = amp * exp(-alpha*|x-c|^2) * dir evaluated on the
 * device (fem.gaussian_source, fem.py:360-364, is amp=-1, alpha=400,
 * c=(.5,.5,.5), dir=(1,1,1)). */
int mdd_assemble_rhs_gaussian(mdd_space* sp, const double* center, double alpha,
                              double amp, const double* dir, mdd_complex* rhs);
/* fem.element_matrices / fem._element_matrices_batch (fem.py:177-207):
 * coords (nt,4,3), signs (nt,6) as doubles; outputs (nt,6,6), (nt,6,6), (nt). */
int mdd_element_matrices(mdd_ctx* ctx, int64_t nt, const double* coords,
                         const double* signs, double* s_el, double* m_el, double* vol);

/* Second-order Nedelec fine space (BASELINE.json config 2; no reference
 * counterpart: the reference implements Whitney elements only, fem.py:1-7).
 * 20 hierarchical basis functions per tet, defined with the tet's vertices
 * sorted by global index: 6 Whitney, 6 edge gradients grad(l_a l_b), 8 face
 * functions (l_c w_ab, l_a w_bc per face (a<b<c)); tet_dofs (nt,20) gives the
 * global DoF of each (-1 = eliminated by PEC).  qbary (nq,4) / qweights (nq)
 * are the load-vector quadrature (weights sum to 1).  mdd_assemble /
 * mdd_assemble_rhs* accept the returned space (PEC only); for
 * mdd_assemble_rhs the source values are laid out (nq, nt, 3). */
int mdd_space2_create(mdd_ctx* ctx, int32_t cells_per_axis, int64_t nv, const double* vertices,
                      int64_t nt, const int64_t* tets, const int64_t* tet_dofs, int64_t ndof,
                      int32_t nq, const double* qbary, const double* qweights, mdd_space** out);
/* 20x20 element matrices of the order-2 basis for tets given by coords (nt,4,3)
 * (vertex order = basis frame). */
int mdd_element2_matrices(mdd_ctx* ctx, int64_t nt, const double* coords, double* s_el, double* m_el);

/* -------------------------------------------- decomposition (host C++)
 * Setup-time index work of reference decomp.py / mesh.py (SURVEY.md §8f rank
 * 1), threaded C++ over the structured Kuhn mesh; no device needed.  Arrays
 * returned through out-pointers are malloc'ed by the library: release them
 * with mdd_free.  Index sets are bit-identical to the reference's. */
void mdd_free(void* p);
/* decomp.extend_overlap (decomp.py:97-110): nsub tet sets (part_ptr/part_idx)
 * grown by `layers` rings of vertex-touching tets; outputs ascending. */
int mdd_extend_overlap(int32_t cells_per_axis, int64_t nv, const int64_t* tets, int32_t nsub,
                       const int64_t* part_ptr, const int64_t* part_idx, int32_t layers,
                       int64_t** out_ptr, int64_t** out_idx);
/* decomp.subdomain_dof_sets (decomp.py:140-176); tet_faces != NULL selects the
 * order-2 space (face DoFs, numbering [e | e+ned | f+2ned | f+2ned+nfd]). */
int mdd_subdomain_dofs(int32_t cells_per_axis, int64_t nv, const int64_t* tets, const int64_t* tet_edges,
                       int64_t ne, const int64_t* edge_to_dof, int64_t ned, const int64_t* tet_faces, int64_t nf,
                       const int64_t* face_to_dof, int64_t nfd, int32_t nsub, const int64_t* sub_ptr,
                       const int64_t* sub_tets, int64_t** out_ptr, int64_t** out_dofs);
/* mesh.nesting_map (mesh.py:231-263): out[nt_fine] = containing coarse tet. */
int mdd_nesting_map(int32_t nc, const double* cverts, const int64_t* ctets, int32_t nf, const double* fverts,
                    const int64_t* ftets, double tol, int64_t* out);
/* decomp.coarse_restriction for nested meshes (decomp.py:212-297): R0 as CSR
 * (ncs rows over the nkept fine DoFs); *bad_edge = fine edge of a
 * tangential-trace discontinuity (MDD_EDECOMP). */
int mdd_coarse_restriction(int64_t nv, const double* fverts, int64_t ntf, const int64_t* ftet_edges,
                           const int64_t* fedges, int64_t nkept, const int64_t* kept_edges, const double* cverts,
                           int64_t ntc, const int64_t* ctets, const int64_t* ctet_edges, const int64_t* csigns,
                           const int64_t* cedge_to_dof, int64_t ncs, const int64_t* tet_map, double continuity_tol,
                           int64_t** out_rowptr, int64_t** out_cols, double** out_vals, int64_t* bad_edge);

/* ------------------------------------------------------ preconditioner
 * precond.PreconditionerState.__init__ / setup (precond.py:150-193, 250-257)
 * and PreconditionerState.apply (precond.py:217-245).
 *
 * Subdomain local problems are factorised by a batched multifrontal
 * elimination over a geometric nested-dissection ordering (replaces the
 * DenseLU/zgetrf of linalg.py:73-107); the coarse block R0 A R0^T is formed by
 * an element-wise Galerkin kernel and factorised the same way. */
typedef struct {
  int family;      /* 0 as, 1 ras, 2 impras   (precond.py:42)               */
  int levels;      /* 1 or 2                                                 */
  int correction;  /* 0 additive, 1 hybrid, 2 adef1 (precond.py:43)         */
  int64_t lu_cap;  /* SizeCapError threshold on a local block, <=0: none     */
  int leaf_size;   /* nested-dissection leaf size (0 -> default)             */
  /* fine level */
  const mdd_csr* A_prec;  /* assembled at xi_prec (precond.py:155-157)       */
  const mdd_csr* A_corr;  /* matrix inside hybrid/adef1 (precond.py:159)     */
  int32_t nsub;
  const int64_t* sub_ptr;   /* nsub+1 offsets into sub_dofs                  */
  const int64_t* sub_dofs;  /* sorted global DOF sets I_l (decomp.py:140-191) */
  const double* sub_pou;    /* aligned weights (decomp.py:194-205) or NULL   */
  const int32_t* dof_xyz;   /* (ndof,3) DoF positions in 1/dof_grid cell units */
  /* impras: local matrices assembled on the submesh (precond.py:82-139)    */
  const mdd_space* space;   /* fine lowest-order space (impras local assembly,
                               coarse Galerkin; for an order-2 fine space its
                               Whitney companion on the same mesh)            */
  const mdd_coeffs* prec_coeffs;
  const int64_t* sub_tet_ptr; /* nsub+1 offsets into sub_tets (impras)        */
  const int64_t* sub_tets;    /* per-subdomain tet lists (decomp.elements)    */
  const int64_t* sub_bface_ptr; /* nsub+1 offsets (impras boundary faces)     */
  const int64_t* sub_bfaces;    /* (.,3) sorted vertex triples                */
  /* coarse level (levels == 2) */
  const mdd_csr* R0;          /* (ncs x ndof) real, decomp.py:212-297        */
  const mdd_space* coarse_space;
  const int64_t* tet_map;     /* fine tet -> coarse tet (mesh.py:231-263)    */
  const int32_t* coarse_dof_xyz; /* (ncs,3) half-cell units of the coarse mesh */
  int64_t nbf_global;         /* global impedance faces (bc=impedance) or 0  */
  const int64_t* bfaces_global;
  int32_t dof_grid;           /* dof_xyz units per mesh cell: 2 (edge midpoints,
                                 0 = default) or 6 (order-2 edges and faces)  */
} mdd_prec_desc;

/* On MDD_ESINGULAR/MDD_ECAP, *failed_ctx is the subdomain id, or -1 for the
 * coarse space. */
int mdd_prec_create(mdd_ctx* ctx, const mdd_prec_desc* desc, mdd_prec** out,
                    int32_t* failed_ctx);
/* PreconditionerState.variant (precond.py:195-213): a view sharing factors. */
int mdd_prec_variant(const mdd_prec* base, int family, int levels, int correction,
                     const mdd_csr* A_corr, mdd_prec** out);
void mdd_prec_destroy(mdd_prec* P);
int mdd_prec_apply(mdd_prec* P, const mdd_complex* v, mdd_complex* out);
/* PreconditionerState.coarse_solve (precond.py:227-228): R0^T A0^{-1} R0 v */
int mdd_prec_coarse_apply(mdd_prec* P, const mdd_complex* v, mdd_complex* out);
/* Diagnostics: device-timed applies (inputs resident, CUDA events on the
 * context stream).  which: 0 full apply, 1 restriction + subdomain solves,
 * 2 coarse solve.  No reference counterpart (bench.py / tools only). */
int mdd_prec_apply_bench(mdd_prec* P, int which, int reps, double* ms_per_call);
/* Multi-GPU sharding (the reference has no distributed code,
 * SPEC.md:8).  Each rank builds its preconditioner over its own block of
 * subdomains (coarse space replicated); attaching a communicator and the row
 * ranges (mdd_prec_set_halo) makes the one-level part of every apply a partial
 * sum completed by a neighbour overlap-sum exchange.  NCCL is resolved with
 * dlopen at first use.  id128 == NULL
 * creates a one-rank communicator without NCCL (collectives are identities);
 * with an id NCCL is initialised even for one rank. */
int mdd_comm_unique_id(char* out128);
int mdd_comm_create(mdd_ctx* ctx, int nranks, int rank, const char* id128, mdd_comm** out);
void mdd_comm_destroy(mdd_comm* c);
int mdd_comm_info(const mdd_comm* c, int* nranks, int* rank);
int mdd_prec_set_comm(mdd_prec* P, mdd_comm* comm);
/* Sharded data plane (no reference counterpart).  Rank q owns the rows
 * [q*ceil(n/N), (q+1)*ceil(n/N)) of every vector and needs the rows [need_lo, need_hi)
 * (the unknowns of its subdomains, reference precond.py:220, and the columns of its rows
 * of A, krylov.py:95-97; contiguous because the reference numbering is x-major and a
 * rank's subdomain block is an x-slab).  After this call the collectives of an apply are:
 *   prolongation overlap sums  - neighbour ncclSend/ncclRecv of the ghost rows, owner adds
 *                                (reference precond.py:224, `out[dofs] += u`);
 *   halo for SpMV/restriction  - neighbour ncclSend/ncclRecv of owned rows, in place;
 *   coarse restriction         - local product with R0 restricted to the owned columns
 *                                + ncclAllReduce of the ncs coarse values (reference
 *                                precond.py:227-228); the coarse solve is replicated.
 * No collective moves a whole vector. */
int mdd_prec_set_halo(mdd_prec* P, int64_t need_lo, int64_t need_hi);
int mdd_prec_halo_info(const mdd_prec* P, int64_t* own_lo, int64_t* own_hi, int64_t* need_lo, int64_t* need_hi,
                       int64_t* exchanged_rows);
/* Loopback group (test infrastructure for the multi-rank path on ONE GPU;
 * no reference counterpart): nranks (<= 8) host threads, each with its own
 * context on the same device, join one group; every collective synchronises
 * the caller's stream, meets the other ranks at a host barrier and moves the
 * data with device copies (allreduce: each rank sums all ranks' buffers in
 * rank order).  Kernels never wait on other ranks, only host threads do. */
int mdd_comm_loopback_group(int nranks, void** group_out);
void mdd_comm_loopback_group_free(void* group);
int mdd_comm_create_loopback(mdd_ctx* ctx, void* group, int rank, mdd_comm** out);
/* marks a loopback group as failed: every rank's current and later collectives return MDD_ENCCL at once */
int mdd_comm_abort(mdd_comm* c);

/* precond.assemble_local(space, coeffs, elems, local_bc="impedance") (precond.py:82-139): the
 * submesh matrix of one subdomain of an impras preconditioner as the device assembled it
 * (element scatter over the subdomain tets + impedance mass over its boundary faces), CSR over
 * the subdomain's unknowns in ascending global order. */
int mdd_prec_local_matrix_size(const mdd_prec* P, int32_t sub, int64_t* n, int64_t* nnz);
int mdd_prec_local_matrix(const mdd_prec* P, int32_t sub, int32_t* rowptr, int32_t* cols, mdd_complex* vals);
/* Smallest pivot ratio min|pivot| / max|pivot| of the last factorisation (subdomain blocks,
 * coarse block).  The reference's DenseLU pivots partially and checks 1e-14 (linalg.py:92-101);
 * the device factorisation pivots statically, which Lemma 2.5 of the paper covers when the
 * problem has absorption or impedance terms.  Without either (xi_prec = 0, sigma = 0, PEC
 * local problems) the caller uses this ratio to refuse an unreliable factor. */
int mdd_prec_pivot_ratio(const mdd_prec* P, double* sub_ratio, double* coarse_ratio);
/* statistics: [n_fronts, max_front, factor_entries, factor_flops, setup_ms,
 *              levels, sum_local_dofs, coarse_n] */
int mdd_prec_stats(const mdd_prec* P, double* out8);
/* Real flop counts of one numeric factorisation (subdomain blocks + coarse block):
 * [0] 8 np m^2 summed over the fronts (full Gauss-Jordan elimination of every front, the figure
 *     mdd_prec_stats reports), [1] what a partial LU of the same fronts needs (the zgetrf the
 *     reference calls, linalg.py:92), [2] what the kernels executed in the last factorisation
 *     (pivot-block inverse + F_PU / Schur GEMMs; a symmetric A_prec skips the F_UP GEMM and the
 *     Schur tiles above the diagonal). */
int mdd_prec_flop_counts(const mdd_prec* P, double* out3);
/* 1 if the last factorisation found A_prec bitwise complex symmetric and
 * formed the packed F_UP blocks as F_PU^T (no second GEMM), else 0 */
int mdd_prec_symmetric(const mdd_prec* P, int* sym);
/* refactorise in place (same pattern) from new A_prec values: the numeric part
 * of setup, used by the benchmark's timed step */
int mdd_prec_refactor(mdd_prec* P, const mdd_csr* A_prec, const mdd_coeffs* prec_coeffs);

/* ------------------------------------------------------------------ GMRES
 * krylov.gmres (krylov.py:64-209): unrestarted GMRES, MGS + one
 * reorthogonalisation pass, complex Givens rotations, right/left
 * preconditioning, optional Hermitian positive definite weight D. */
typedef int (*mdd_host_op)(void* user, int64_t n, const mdd_complex* in, mdd_complex* out);

typedef struct {
  double tol;
  int32_t maxit;
  int32_t side;          /* 0 right, 1 left                                   */
  int32_t check_drift;   /* 1: compute the orthogonality drift (krylov.py:152) */
  int32_t keep_basis;
  int32_t device_io;     /* 1: b, x0, x are device pointers (no H2D/D2H)      */
  int32_t ortho;         /* 0: MGS2 (reference krylov.py:137-143, default);
                            1: CGS2 (classical Gram-Schmidt + one
                            reorthogonalisation pass; with a sharded
                            preconditioner the Krylov vectors are sharded by
                            row blocks over the ranks)                        */
} mdd_gmres_cfg;

typedef struct {
  /* operator: exactly one of A / a_fn */
  const mdd_csr* A;
  mdd_host_op a_fn; void* a_user;
  /* preconditioner: P, m_fn or neither */
  mdd_prec* P;
  mdd_host_op m_fn; void* m_user;
  const mdd_csr* Mcsr;   /* preconditioner given as a matrix */
  /* weight: D (CSR) or NULL */
  const mdd_csr* D;
} mdd_gmres_ops;

int mdd_gmres(mdd_ctx* ctx, const mdd_gmres_ops* ops, int64_t n,
              const mdd_complex* b, const mdd_complex* x0 /* NULL = zero */,
              const mdd_gmres_cfg* cfg,
              mdd_complex* x, double* history /* maxit+1 */,
              double* drift /* maxit+1, NULL ok */, mdd_complex* basis /* (maxit+1)*n or NULL */,
              int32_t* iterations, int32_t* converged, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* MDD_H */
