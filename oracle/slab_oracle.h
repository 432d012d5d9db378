/*
 * slab_oracle.h — C interface of the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY. This is a CPU restatement of the reference's
 * arithmetic for the MG-preconditioned CG hot path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker / the timed CPU baseline. The product
 * path (paper_2304_08232_b200/csrc) never links, loads or calls it.
 *
 * Parity status: PINNED. The oracle is compared bit-for-bit with the real
 * reference headers compiled into oracle/_ref/libslab_ref.so (same C
 * interface, see ref_shim.cpp) and with the golden vectors in tests/golden/
 * that were generated from those headers (tests/golden/make_golden.py).
 *
 * The same declarations are implemented twice:
 *   oracle/slab_oracle.c  -> oracle/libslab_oracle.so   (restatement, kind "port")
 *   oracle/ref_shim.cpp   -> oracle/_ref/libslab_ref.so (reference headers, kind "reference")
 */
#ifndef SLAB_ORACLE_H
#define SLAB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes shared with the GPU C-ABI (reference error.hpp:25-42) */
enum {
	SO_OK = 0,
	SO_DIMENSION_MISMATCH = 1,
	SO_INVALID_ARGUMENT = 2,
	SO_SOLVER_BREAKDOWN = 3
};

typedef struct so_level so_level; /* one ProblemLevel and its coarser chain */

/* which implementation answers: "port" or "reference" */
const char * so_kind( void );
void so_set_threads( int threads ); /* 0 = OpenMP default */
int so_get_threads( void );

/* ---- problem generation (problem.hpp) ---- */
uint64_t so_stencil_nnz( uint64_t nx, uint64_t ny, uint64_t nz );
int so_build_stencil( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * row_offsets, uint64_t * cols, double * vals );
int so_build_restriction_cols( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * cols );

/* ---- rng (rng.hpp) ---- */
uint64_t so_lcg_fill( uint64_t seed, double * out, uint64_t n ); /* returns the state afterwards */
uint64_t so_lcg_next( uint64_t state );

/* ---- primitives on raw arrays (operations.hpp) ---- */
double so_dot( const double * x, const double * y, uint64_t n );
void so_waxpby( double * w, double alpha, const double * x, double beta, const double * y, uint64_t n );
void so_mxv_csr( double * y, uint64_t nrows, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	const double * x );
void so_mxv_csr_masked( double * y, const uint64_t * members, uint64_t nmembers, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x );
void so_mxv_csr_transpose( double * y, uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x );
void so_mxv_csr_transpose_masked( double * y, const uint64_t * members, uint64_t nmembers, uint64_t nrows, uint64_t ncols,
	const uint64_t * row_offsets, const uint64_t * cols, const double * vals, const double * x );

/* ---- levels (problem.hpp ProblemLevel / build_hierarchy, coloring.hpp greedy_color) ---- */
int so_hierarchy_create( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels, so_level ** out );
int so_level_from_csr( uint64_t n, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	so_level ** out );
void so_level_destroy( so_level * level );
so_level * so_level_coarser( so_level * level ); /* NULL at the coarsest */
uint64_t so_level_n( const so_level * level );
uint64_t so_level_nnz( const so_level * level );
void so_level_dims( const so_level * level, uint64_t dims[ 3 ] );
uint64_t so_level_num_colors( const so_level * level );
uint64_t so_level_color_size( const so_level * level, uint64_t k );
uint64_t so_level_color_nnz( const so_level * level, uint64_t k );
void so_level_color_members( const so_level * level, uint64_t k, uint64_t * out );
void so_level_csr( const so_level * level, uint64_t * row_offsets, uint64_t * cols, double * vals );
void so_level_diag( const so_level * level, double * out );
uint64_t so_level_nnz_visited( const so_level * level );
void so_level_reset_stats( so_level * level );
int so_level_mxv( so_level * level, double * y, const double * x ); /* y = A x */

/* ---- smoother / multigrid / cg (smoother.hpp, multigrid.hpp, cg.hpp) ---- */
int so_rbgs_color_step( so_level * level, uint64_t k, double * z, const double * r );
int so_rbgs_forward( so_level * level, double * z, const double * r );
int so_rbgs_backward( so_level * level, double * z, const double * r );
int so_rbgs_symmetric( so_level * level, double * z, const double * r, uint64_t sweeps );
int so_restrict_vector( so_level * level, const double * v_fine, double * out );
int so_refine_and_add( so_level * level, double * z, const double * z_c );
int so_mg_vcycle( so_level * level, double * z, const double * r, uint64_t sweeps );

typedef struct so_cg_config {
	uint64_t max_iters;        /* CGConfig::max_iters, default 500 */
	double rtol;               /* default 1e-6 */
	int use_preconditioner;    /* default 1 */
	int has_fixed_iterations;  /* std::optional engaged? */
	uint64_t fixed_iterations;
	uint64_t sweeps;           /* SmootherConfig::sweeps, default 1 */
} so_cg_config;

/* history must hold max_iters+1 doubles; x receives the solution */
int so_cg_solve( so_level * hierarchy, const double * b, const double * x0, const so_cg_config * cfg, double * x,
	double * history, uint64_t * iterations, int * converged );
int so_residual_norm( so_level * level, const double * x, const double * b, double * out );

#ifdef __cplusplus
}
#endif

#endif
