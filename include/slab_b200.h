/*
 * slab_b200.h — C ABI of the B200-native (sm_100a) implementation of the slab /
 * GraphBLAS-HPCG hot path: the multigrid-preconditioned conjugate-gradient solve on
 * the 27-point stencil.
 *
 * The reference ("slab", /root/reference/proj/include/slab) is a header-only C++20
 * template library with no FFI of its own, so this boundary is *designed*: every entry
 * point below replaces one free function / container of the reference's operator API and
 * cites it as file:line relative to /root/reference/proj/include/slab/. A maintainer binds
 * these through the C++ facade include/slab_b200.hpp (same names, arguments and
 * exceptions as the reference) — see INTEGRATION.md.
 *
 * Conventions
 *  - plain pointers, sizes and opaque handles only; no CUDA or torch types;
 *  - every call returns a status code (0 = ok); codes 1..3 map 1:1 to the reference's
 *    exception taxonomy (error.hpp:25-42) and the facade re-throws them;
 *    slab_last_error() returns the message of the calling thread's last failure;
 *  - all argument checks run before any work, so a failed call leaves outputs untouched;
 *  - containers live in HBM in an opaque format; host access is explicit upload/download
 *    in the reference's natural (x-fastest) ordering;
 *  - one context = one device + one stream; calls are asynchronous on that stream except
 *    those that return data to the host. A context is driven by one host thread at a time
 *    (operations.hpp:27-31: parallelism lives inside the primitives). Several contexts may be
 *    driven by several threads concurrently; what they share process-wide is the launch counter
 *    (atomic) and the tuning knobs of slab_set_tuning / slab_set_programmatic_launch, which are a
 *    benchmarking interface: set them while no other thread is inside the library (they are read
 *    without locks, and changing one invalidates every context's cached graphs at its next use);
 *  - there is NO CPU fallback: creating a context without a usable sm_100 GPU fails with
 *    SLAB_ERR_CUDA.
 */
#ifndef SLAB_B200_H
#define SLAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLAB_B200_ABI_VERSION 1

typedef enum slab_status {
	SLAB_OK = 0,
	SLAB_ERR_DIMENSION_MISMATCH = 1, /* slab::DimensionMismatch  error.hpp:30 */
	SLAB_ERR_INVALID_ARGUMENT = 2,   /* slab::InvalidArgument    error.hpp:35 */
	SLAB_ERR_SOLVER_BREAKDOWN = 3,   /* slab::SolverBreakdown    error.hpp:40 */
	SLAB_ERR_CUDA = 4,               /* CUDA / NCCL runtime failure, or no GPU */
	SLAB_ERR_INTERNAL = 5
} slab_status;

typedef struct slab_ctx_s * slab_ctx_t;     /* device + stream (+ process grid) */
typedef struct slab_vec_s * slab_vec_t;     /* slab::DenseVector   dense_vector.hpp:33-66 */
typedef struct slab_mat_s * slab_mat_t;     /* slab::SparseMatrix  sparse_matrix.hpp:48-171 */
typedef struct slab_mask_s * slab_mask_t;   /* slab::IndexMask     index_mask.hpp:35-73 */
typedef struct slab_level_s * slab_level_t; /* slab::ProblemLevel  problem.hpp:220-277 */

/* slab::Descriptor (descriptor.hpp:26-38) as bit flags */
#define SLAB_DESC_NONE 0u
#define SLAB_DESC_STRUCTURAL 1u
#define SLAB_DESC_TRANSPOSE 2u

/* how dot() reduces (operations.hpp:61-91) */
#define SLAB_DOT_EXACT 0 /* 4096-element chunks summed left to right, partials in chunk order: bit-identical to the reference */
#define SLAB_DOT_TREE 1  /* fixed-shape warp-shuffle/block tree: run-to-run deterministic, differs from the reference by rounding only */

/* ------------------------------------------------------------------ library */
int slab_abi_version( void );
const char * slab_last_error( void );
const char * slab_status_name( int status );
/* number of kernels this library has launched in this process (bench.py's gpu_launches) */
uint64_t slab_launch_count( void );
/* chain kernels with programmatic dependent launch (griddepcontrol): 1 (default) or 0. Process-wide. */
int slab_set_programmatic_launch( int enabled );
/* performance knobs that never change results: "stream_rows" (launches with at least this many rows
 * use the streaming kernel shape), "stream_variant" (which streaming shape), "pdl", "halo_overlap" (boundary
 * rows first, halo messages beside the interior rows), "l2_window"; "planes" / "plane_min_rows" / "plane_ty" /
 * "plane_cz" / "plane_ns" / "plane_autotune" (levels time the tile shapes their cost models propose when they are built) /
 * "plane_warp_sync" / "plane_pad_lines" (plane-phase smoother of regular box levels, csrc/plane.cu), "fuse_rz" (tree-dot
 * mode: r'z on the last plane phases of the V-cycle), "side_rr" (exact-dot mode: r'r on a side stream), "lazy_x" (fixed-iteration
 * solves take the x update one iteration late on a low-priority stream under the coarse levels of the next V-cycle: 0 off,
 * 1 for systems of at least 2^20 rows, 2 always; "lazy_x_prio", "lazy_x_blocks" shape that pass), "iter_batch" (CG iterations per graph launch in
 * fixed-iteration solves: the largest divisor of the iteration count up to this, default 50), "inline_record" (those solves
 * write the history from the p update and count iterations in the r update instead of a bookkeeping launch), "dot_cpb" /
 * "dot_tile" (shape of the exact dot) and "spmv_planes" /
 * "spmv_plane_min_rows" / "spmv_plane_ty" / "spmv_plane_cz" / "spmv_plane_ns" (slab-staged product, csrc/plane_spmv.cu); for the dictionary-coded matrix copy: "packed" (use it, default 1),
 * "pack_build" (build it when a matrix is created, default 1), "keep_plain" (default 1; 0 frees the plain arrays of
 * matrices created afterwards whose coded copy has no escaped rows — 32 instead of 324 bytes per 27-point row, at the
 * price of download / transpose for those matrices), "packed_min_rows" (smaller launches use the plain arrays), "packed_batch", "packed_block", "packed_rows" / "packed_rows_spmv" (rows per thread of
 * colour steps / products), "packed_multi_min_rows"; "cluster_rows" (default 384: levels whose largest
 * colour has at most this many rows run a whole symmetric sweep as ONE launch, csrc/sweep_cluster.cu — one CTA up to 512
 * rows, a thread-block cluster up to 4096, which is an experiment that does not pay; 0 = per-colour launches; env SLAB_CLUSTER_ROWS). Process-wide; each also has an environment variable
 * SLAB_<KEY> for the first four packed keys and the older ones. */
int slab_set_tuning( const char * key, int64_t value );
/* Environment only: SLAB_PLANE_TUNE_CACHE=<file> keeps the tile shapes the plane phases measured ("lx ly lz phase ty cz
 * ns" per line) and re-uses them in later processes — a run and a profiler's run of it then execute the same shapes;
 * SLAB_PLANE_DEBUG=1 prints the shapes. */

/* ------------------------------------------------------------------ context */
int slab_ctx_create( int device, slab_ctx_t * out );
int slab_ctx_destroy( slab_ctx_t ctx );
int slab_ctx_sync( slab_ctx_t ctx );
int slab_ctx_set_dot_mode( slab_ctx_t ctx, int mode ); /* SLAB_DOT_EXACT (default) | SLAB_DOT_TREE */
int slab_ctx_get_dot_mode( slab_ctx_t ctx, int * mode );
/* use CUDA graphs for the V-cycle / CG iteration (default 1) */
int slab_ctx_set_graphs( slab_ctx_t ctx, int enabled );
/* fuse residual+restriction and prolongation+update (default 1); 0 runs the reference's
 * primitive-by-primitive composition (multigrid.hpp:100-104, :76-77) */
int slab_ctx_set_fused_transfers( slab_ctx_t ctx, int enabled );
/* LevelStats timing (problem.hpp:204-209, the monotonic_ns wrappers of smoother.hpp:79-98 and
 * multigrid.hpp:50-53,75-79,92-114): when enabled, V-cycles run launch by launch with CUDA events around the
 * same sections, and smoother_ns / transfer_ns / mg_ns are filled (device time). Off by default: the fast
 * path replays CUDA graphs, where only nnz_visited is maintained. */
int slab_ctx_set_profiling( slab_ctx_t ctx, int enabled );
/* device-side elapsed time between two marks on the context's stream, milliseconds */
int slab_ctx_timer_start( slab_ctx_t ctx );
int slab_ctx_timer_stop( slab_ctx_t ctx, double * elapsed_ms );
int slab_ctx_device_info( slab_ctx_t ctx, int * sm_count, int * cc_major, int * cc_minor, uint64_t * hbm_bytes );

/* ------------------------------------------------------------------ vectors (dense_vector.hpp, operations.hpp) */
int slab_vec_create( slab_ctx_t ctx, uint64_t n, double value, slab_vec_t * out ); /* DenseVector(n, value) :37 */
int slab_vec_destroy( slab_vec_t v );
int slab_vec_size( slab_vec_t v, uint64_t * n );                              /* size() :45 */
int slab_vec_upload( slab_vec_t v, const double * host, uint64_t n );        /* DenseVector::from :39 */
int slab_vec_download( slab_vec_t v, double * host, uint64_t n );            /* values() :56 */
int slab_vec_copy( slab_vec_t dst, slab_vec_t src );                         /* copy assignment */
int slab_vec_fill_lcg( slab_vec_t v, uint64_t seed, uint64_t * state_out );  /* random_vector rng.hpp:59-65 (host LCG, then upload) */

int slab_set_all( slab_vec_t v, double value );                              /* set_all operations.hpp:49-54 */
int slab_dot( slab_vec_t x, slab_vec_t y, double * out );                    /* dot operations.hpp:61-91 */
int slab_waxpby( slab_vec_t w, double alpha, slab_vec_t x, double beta, slab_vec_t y ); /* waxpby operations.hpp:97-106 */

/* ------------------------------------------------------------------ matrices (sparse_matrix.hpp, problem.hpp) */
/* SparseMatrix::from_csr sparse_matrix.hpp:96-124 — same validation, 64-bit indices in */
int slab_mat_create_csr( slab_ctx_t ctx, uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets,
	const uint64_t * col_indices, const double * values, slab_mat_t * out );
/* build_matrix problem.hpp:90-131 — generated on the device, no host CSR */
int slab_mat_create_stencil27( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, slab_mat_t * out );
/* build_restriction problem.hpp:174-201 */
int slab_mat_create_restriction( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, slab_mat_t * out );
int slab_mat_destroy( slab_mat_t A );
int slab_mat_shape( slab_mat_t A, uint64_t * nrows, uint64_t * ncols, uint64_t * nnz ); /* nrows/ncols/nnz :126-134 */
/* row_offsets()/col_indices()/values() :136-144 — converts the opaque format back to CSR */
int slab_mat_download_csr( slab_mat_t A, uint64_t * row_offsets, uint64_t * col_indices, double * values );
/* bytes the opaque format occupies in HBM (values + indices + slice table) */
int slab_mat_device_bytes( slab_mat_t A, uint64_t * bytes );
/* How the matrix is held on the device. Every matrix has the plain SELL-32 arrays (12 bytes per stored
 * entry); matrices with few distinct (column - row, value) pairs also get a dictionary-coded copy (1 byte
 * per entry) that the kernels read instead — same arithmetic, same order, same bits. */
typedef struct slab_format_info {
	int32_t packed;         /* 1 when the dictionary-coded copy exists */
	int32_t width_class;    /* codes per row the kernels are instantiated for (>= widest row), 0 if not packed */
	int32_t dict_size;      /* dictionary entries in use (entry 0 = padding) */
	int32_t stride;         /* slices between rows that mostly repeat their codes (multi-row kernels), 0 = none */
	int64_t escaped_rows;   /* rows with an entry outside the dictionary: read from the plain arrays */
	uint64_t plain_bytes;   /* bytes of the plain arrays */
	uint64_t packed_bytes;  /* bytes of the coded copy */
	uint64_t mask_bytes;    /* bytes of the 27-offset row masks (4 per row) that the shared-memory-staged kernels read on
	                           box-shaped levels of a single-process context; 0 when the matrix has none */
	int32_t plane_phases;   /* 1 when the matrix is a regular 27-point box operator (one value per offset, every row
	                           storing exactly its in-box offsets): sweeps and products then run from zero-padded
	                           plane slabs in shared memory and read no matrix stream at all */
	int32_t reserved;
} slab_format_info;
int slab_mat_format_info( slab_mat_t A, slab_format_info * out );

/* ------------------------------------------------------------------ masks (index_mask.hpp) */
int slab_mask_create( slab_ctx_t ctx, uint64_t universe, const uint64_t * members, uint64_t count,
	slab_mask_t * out );                                                      /* IndexMask(universe, members) :39-49 */
int slab_mask_destroy( slab_mask_t m );
int slab_mask_info( slab_mask_t m, uint64_t * universe, uint64_t * count );

/* mxv operations.hpp:213-218 (unmasked) and :225-230 (masked); desc = SLAB_DESC_* flags.
 * Same checks as mxv_checked :147-160, including the &y == &x aliasing rejection. */
int slab_mxv( slab_vec_t y, slab_mat_t A, slab_vec_t x, unsigned desc );
int slab_mxv_masked( slab_vec_t y, slab_mask_t mask, slab_mat_t A, slab_vec_t x, unsigned desc );

/* ------------------------------------------------------------------ levels (problem.hpp, coloring.hpp) */
/* build_hierarchy problem.hpp:284-319: the whole chain is generated on the device */
int slab_hierarchy_create( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels,
	slab_level_t * out );
/* ProblemLevel(SparseMatrix) problem.hpp:253 — standalone level around an arbitrary square
 * system given as CSR: extract_diagonal :143-166 + greedy_color coloring.hpp:114-158 (host, setup only) */
int slab_level_create_csr( slab_ctx_t ctx, uint64_t n, const uint64_t * row_offsets, const uint64_t * col_indices,
	const double * values, slab_level_t * out );
int slab_level_destroy( slab_level_t level ); /* destroys the coarser chain too */
int slab_level_coarser( slab_level_t level, slab_level_t * out ); /* NULL handle at the coarsest */
int slab_level_matrix( slab_level_t level, slab_mat_t * A );      /* borrowed: level.A */
int slab_level_restriction( slab_level_t level, slab_mat_t * R ); /* borrowed: *level.restriction, NULL at the coarsest */
int slab_level_diag( slab_level_t level, slab_vec_t * a_diag );   /* borrowed: level.a_diag */
int slab_level_info( slab_level_t level, uint64_t dims[ 3 ], uint64_t * n, uint64_t * nnz, uint64_t * num_colors,
	uint64_t * depth );
int slab_level_color_info( slab_level_t level, uint64_t k, uint64_t * size, uint64_t * color_nnz );
int slab_level_color_members( slab_level_t level, uint64_t k, uint64_t * members ); /* colors.masks[k].members() */

typedef struct slab_level_stats { /* LevelStats problem.hpp:204-209; times from CUDA events */
	uint64_t smoother_ns;
	uint64_t transfer_ns;
	uint64_t mg_ns;
	uint64_t nnz_visited;
} slab_level_stats;
int slab_level_stats_get( slab_level_t level, slab_level_stats * out );
/* format of the level's colour-major matrix copy (the one the smoother reads) */
int slab_level_format_info( slab_level_t level, slab_format_info * out );
int slab_level_stats_reset( slab_level_t level ); /* reset_stats problem.hpp:271-276 */

/* ------------------------------------------------------------------ smoother (smoother.hpp) */
int slab_rbgs_color_step( slab_level_t level, uint64_t k, slab_vec_t z, slab_vec_t r ); /* rbgs_color_step :60-72, fused */
/* the same step twice in a row as ONE launch — what rbgs_symmetric does at the turnaround between its forward and
 * backward sweep (:108-111: the last colour runs twice). Bit-identical to two calls of slab_rbgs_color_step; on a
 * decomposed level the colour's halo message goes out once, after the second update. */
int slab_rbgs_color_step_twice( slab_level_t level, uint64_t k, slab_vec_t z, slab_vec_t r );
int slab_rbgs_forward( slab_level_t level, slab_vec_t z, slab_vec_t r );               /* :77-85 */
int slab_rbgs_backward( slab_level_t level, slab_vec_t z, slab_vec_t r );              /* :92-100 */
int slab_rbgs_symmetric( slab_level_t level, slab_vec_t z, slab_vec_t r, uint64_t sweeps ); /* :103-113 */

/* ------------------------------------------------------------------ multigrid (multigrid.hpp) */
int slab_restrict_vector( slab_level_t level, slab_vec_t v_fine, slab_vec_t out ); /* :46-54 */
int slab_refine_and_add( slab_level_t level, slab_vec_t z, slab_vec_t z_c );       /* :71-81 */
int slab_mg_vcycle( slab_level_t level, slab_vec_t z, slab_vec_t r, uint64_t sweeps ); /* :87-116 */

/* ------------------------------------------------------------------ cg (cg.hpp) */
typedef struct slab_cg_config { /* CGConfig cg.hpp:41-48 + SmootherConfig smoother.hpp:48-50 */
	uint64_t max_iters;       /* 500 */
	double rtol;              /* 1e-6 */
	int use_preconditioner;   /* 1 */
	int has_fixed_iterations; /* 0 */
	uint64_t fixed_iterations;
	uint64_t sweeps;          /* 1 */
} slab_cg_config;
void slab_cg_config_default( slab_cg_config * cfg );

typedef struct slab_cg_result { /* CGResult cg.hpp:50-56 (the solution is the x vector) */
	uint64_t iterations;
	int converged;
	double solve_ms; /* device time of the solve, CUDA events on the context's stream */
} slab_cg_result;

/* cg_solve cg.hpp:77-142 on device-resident vectors: x <- x0, then iterate. history must
 * hold min(fixed_iterations, max_iters)+1 (or max_iters+1) doubles. */
int slab_cg_solve( slab_level_t hierarchy, slab_vec_t b, slab_vec_t x0, const slab_cg_config * cfg, slab_vec_t x,
	double * history, slab_cg_result * result );
/* the same call with HOST buffers: uploads b and x0, solves, downloads x (the e2e path) */
int slab_cg_solve_host( slab_level_t hierarchy, const double * b, const double * x0, uint64_t n,
	const slab_cg_config * cfg, double * x, double * history, slab_cg_result * result );
/* residual_norm cg.hpp:59-67 */
int slab_residual_norm( slab_mat_t A, slab_vec_t x, slab_vec_t b, double * out );

/* ------------------------------------------------------------------ 3D domain decomposition (no reference
 * equivalent: distributed execution is out of the reference's scope; the paper's MPI "Ref" exchanges
 * geometric halos per colour). One process per GPU. After slab_ctx_set_process_grid the dims
 * given to slab_hierarchy_create are the LOCAL grid of this rank; the global grid is local x process grid, every
 * level is decomposed the same way, colours and column order follow GLOBAL coordinates so that per-row
 * arithmetic is identical to the single-process solve on the global grid. Vectors created on such a context
 * carry a ghost tail; create them after the hierarchy. dot() returns the sum over ranks once a communicator is
 * attached. Direction index = (dz+1)*9 + (dy+1)*3 + (dx+1). */
int slab_ctx_set_process_grid( slab_ctx_t ctx, int px, int py, int pz, int rank ); /* rank = rx + px*(ry + py*rz) */
int slab_nccl_unique_id( unsigned char * out128 );                /* rank 0 creates it, everybody gets a copy */
int slab_ctx_init_nccl( slab_ctx_t ctx, const unsigned char * id128 ); /* collective: ncclCommInitRank */
int slab_ctx_dist_info( slab_ctx_t ctx, int grid[ 3 ], int * rank, int * nranks, int * has_comm, uint64_t * exchanges );
int slab_level_decomp( slab_level_t level, uint64_t global_dims[ 3 ], uint64_t offset[ 3 ], uint64_t * n_ghost );
/* manual halo access (no communicator attached): what a custom transport or a test moves between ranks.
 * colour -1 = all colours of that direction. pack gathers this rank's boundary values into host_out;
 * unpack stores a peer's packed values into the ghost range of v. */
int slab_level_halo_info( slab_level_t level, int dir, int color, uint64_t * send_count, uint64_t * recv_count, int * peer );
int slab_level_halo_pack( slab_level_t level, slab_vec_t v, int dir, int color, double * host_out );
int slab_level_halo_unpack( slab_level_t level, slab_vec_t v, int dir, int color, const double * host_in );
/* host-only view of the halo plan of any rank (runs without a GPU): counts, peer, first ghost slot and the
 * local indices of the send list of (direction, colour); and the local (owned or ghost) index of a global point */
int slab_plan_query( const uint64_t local_dims[ 3 ], const uint64_t grid[ 3 ], uint64_t rank, int dir, int color,
	uint64_t * n_local, uint64_t * n_ghost, uint64_t * send_count, uint64_t * recv_count, int64_t * peer,
	uint64_t * ghost_base, uint64_t * send_indices );
int slab_plan_local_index( const uint64_t local_dims[ 3 ], const uint64_t grid[ 3 ], uint64_t rank, uint64_t X, uint64_t Y,
	uint64_t Z, int64_t * out );

#ifdef __cplusplus
}
#endif

#endif /* SLAB_B200_H */
