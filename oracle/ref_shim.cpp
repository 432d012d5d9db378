/*
 * ref_shim.cpp — exposes the UNMODIFIED reference headers
 * (/root/reference/proj/include/slab/ *.hpp) through the C interface of
 * slab_oracle.h, so that the restatement in slab_oracle.c can be pinned
 * against the reference itself and so that bench.py can time the reference's
 * own CPU implementation (cpu_baseline.kind = "reference").
 *
 * TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into
 * oracle/_ref/libslab_ref.so when /root/reference is present; the sources stay
 * where they are (only -I points at them), nothing is copied into the repo.
 * This file contains no reference code: it only calls the reference API.
 */
#include "slab_oracle.h"

#include <cstring>
#include <memory>
#include <vector>

#include <slab/cg.hpp>
#include <slab/coloring.hpp>
#include <slab/dense_vector.hpp>
#include <slab/multigrid.hpp>
#include <slab/operations.hpp>
#include <slab/parallel.hpp>
#include <slab/problem.hpp>
#include <slab/rng.hpp>
#include <slab/smoother.hpp>
#include <slab/sparse_matrix.hpp>

using namespace slab;

struct so_level {
	ProblemLevel * level;            // borrowed for coarser links
	std::unique_ptr< ProblemLevel > owner; // set on the head only
	std::unique_ptr< so_level > coarser;
};

namespace {

	int status_of( const std::exception & e ) {
		if( dynamic_cast< const DimensionMismatch * >( &e ) ) {
			return SO_DIMENSION_MISMATCH;
		}
		if( dynamic_cast< const SolverBreakdown * >( &e ) ) {
			return SO_SOLVER_BREAKDOWN;
		}
		return SO_INVALID_ARGUMENT;
	}

	DenseVector vec_from( const double * p, std::size_t n ) {
		return DenseVector::from( std::vector< double >( p, p + n ) );
	}

	void vec_to( const DenseVector & v, double * p ) {
		if( v.size() > 0 ) {
			std::memcpy( p, v.values().data(), v.size() * sizeof( double ) );
		}
	}

	SparseMatrix csr_from( std::size_t nrows, std::size_t ncols, const uint64_t * ro, const uint64_t * co,
		const double * va ) {
		const std::size_t nnz = ro[ nrows ];
		return SparseMatrix::from_csr( nrows, ncols, std::vector< std::size_t >( ro, ro + nrows + 1 ),
			std::vector< std::size_t >( co, co + nnz ), std::vector< double >( va, va + nnz ) );
	}

	so_level * wrap_chain( std::unique_ptr< ProblemLevel > head ) {
		so_level * out = new so_level{};
		out->level = head.get();
		out->owner = std::move( head );
		so_level * at = out;
		while( at->level->has_coarser() ) {
			at->coarser = std::make_unique< so_level >();
			at->coarser->level = at->level->coarser.get();
			at = at->coarser.get();
		}
		return out;
	}

	template< class F >
	int guarded( F && f ) {
		try {
			f();
			return SO_OK;
		} catch( const std::exception & e ) {
			return status_of( e );
		}
	}

} // namespace

extern "C" {

const char * so_kind( void ) {
	return "reference";
}
void so_set_threads( int threads ) {
	set_max_threads( static_cast< unsigned >( threads ) );
}
int so_get_threads( void ) {
	return static_cast< int >( max_threads() );
}

uint64_t so_stencil_nnz( uint64_t nx, uint64_t ny, uint64_t nz ) {
	return stencil_nnz( GridDims{ nx, ny, nz } );
}

int so_build_stencil( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * row_offsets, uint64_t * cols, double * vals ) {
	return guarded( [ & ] {
		const SparseMatrix A = build_matrix( GridDims{ nx, ny, nz } );
		std::memcpy( row_offsets, A.row_offsets().data(), ( A.nrows() + 1 ) * sizeof( uint64_t ) );
		std::memcpy( cols, A.col_indices().data(), A.nnz() * sizeof( uint64_t ) );
		std::memcpy( vals, A.values().data(), A.nnz() * sizeof( double ) );
	} );
}

int so_build_restriction_cols( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * cols ) {
	return guarded( [ & ] {
		const SparseMatrix R = build_restriction( GridDims{ nx, ny, nz } );
		std::memcpy( cols, R.col_indices().data(), R.nnz() * sizeof( uint64_t ) );
	} );
}

uint64_t so_lcg_next( uint64_t state ) {
	Lcg64 rng( state );
	return rng.next_u64();
}

uint64_t so_lcg_fill( uint64_t seed, double * out, uint64_t n ) {
	Lcg64 rng( seed );
	const DenseVector v = random_vector( n, rng );
	vec_to( v, out );
	// recover the state: replay the integer recurrence (next_u64 is the only mutator)
	Lcg64 replay( seed );
	uint64_t state = seed;
	for( uint64_t i = 0; i < n; ++i ) {
		state = replay.next_u64();
	}
	return state;
}

double so_dot( const double * x, const double * y, uint64_t n ) {
	return dot( vec_from( x, n ), vec_from( y, n ) );
}

void so_waxpby( double * w, double alpha, const double * x, double beta, const double * y, uint64_t n ) {
	// honour aliasing the way the reference call sites do (cg.hpp:128-129)
	DenseVector xv = vec_from( x, n );
	if( w == x && w == y ) {
		waxpby( xv, alpha, xv, beta, xv );
		vec_to( xv, w );
	} else if( w == x ) {
		const DenseVector yv = vec_from( y, n );
		waxpby( xv, alpha, xv, beta, yv );
		vec_to( xv, w );
	} else if( w == y ) {
		DenseVector yv = vec_from( y, n );
		waxpby( yv, alpha, xv, beta, yv );
		vec_to( yv, w );
	} else {
		const DenseVector yv = vec_from( y, n );
		DenseVector wv( n );
		waxpby( wv, alpha, xv, beta, yv );
		vec_to( wv, w );
	}
}

void so_mxv_csr( double * y, uint64_t nrows, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	const double * x ) {
	uint64_t ncols = 0;
	for( uint64_t k = 0; k < row_offsets[ nrows ]; ++k ) {
		ncols = cols[ k ] + 1 > ncols ? cols[ k ] + 1 : ncols;
	}
	const SparseMatrix A = csr_from( nrows, ncols, row_offsets, cols, vals );
	DenseVector yv( nrows );
	mxv( yv, A, vec_from( x, ncols ) );
	vec_to( yv, y );
}

void so_mxv_csr_masked( double * y, const uint64_t * members, uint64_t nmembers, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x ) {
	// nrows is not part of this signature: the largest member bounds the rows that matter
	uint64_t nrows = 0;
	for( uint64_t m = 0; m < nmembers; ++m ) {
		nrows = members[ m ] + 1 > nrows ? members[ m ] + 1 : nrows;
	}
	uint64_t ncols = 0;
	for( uint64_t k = 0; k < row_offsets[ nrows ]; ++k ) {
		ncols = cols[ k ] + 1 > ncols ? cols[ k ] + 1 : ncols;
	}
	const SparseMatrix A = csr_from( nrows, ncols, row_offsets, cols, vals );
	const IndexMask mask( nrows, std::vector< std::size_t >( members, members + nmembers ) );
	DenseVector yv = vec_from( y, nrows );
	mxv( yv, mask, A, vec_from( x, ncols ), descriptors::structural );
	vec_to( yv, y );
}

void so_mxv_csr_transpose( double * y, uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x ) {
	const SparseMatrix A = csr_from( nrows, ncols, row_offsets, cols, vals );
	DenseVector yv( ncols );
	mxv( yv, A, vec_from( x, nrows ), descriptors::transpose_matrix );
	vec_to( yv, y );
}

void so_mxv_csr_transpose_masked( double * y, const uint64_t * members, uint64_t nmembers, uint64_t nrows, uint64_t ncols,
	const uint64_t * row_offsets, const uint64_t * cols, const double * vals, const double * x ) {
	const SparseMatrix A = csr_from( nrows, ncols, row_offsets, cols, vals );
	const IndexMask mask( ncols, std::vector< std::size_t >( members, members + nmembers ) );
	DenseVector yv = vec_from( y, ncols );
	mxv( yv, mask, A, vec_from( x, nrows ), descriptors::structural_transpose );
	vec_to( yv, y );
}

int so_hierarchy_create( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels, so_level ** out ) {
	*out = nullptr;
	return guarded( [ & ] {
		auto head = std::make_unique< ProblemLevel >( build_hierarchy( GridDims{ nx, ny, nz }, levels ) );
		*out = wrap_chain( std::move( head ) );
	} );
}

int so_level_from_csr( uint64_t n, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	so_level ** out ) {
	*out = nullptr;
	return guarded( [ & ] {
		auto head = std::make_unique< ProblemLevel >( csr_from( n, n, row_offsets, cols, vals ) );
		*out = wrap_chain( std::move( head ) );
	} );
}

void so_level_destroy( so_level * level ) {
	delete level;
}
so_level * so_level_coarser( so_level * level ) {
	return level->coarser.get();
}
uint64_t so_level_n( const so_level * level ) {
	return level->level->n();
}
uint64_t so_level_nnz( const so_level * level ) {
	return level->level->A.nnz();
}
void so_level_dims( const so_level * level, uint64_t dims[ 3 ] ) {
	dims[ 0 ] = level->level->dims.nx;
	dims[ 1 ] = level->level->dims.ny;
	dims[ 2 ] = level->level->dims.nz;
}
uint64_t so_level_num_colors( const so_level * level ) {
	return level->level->colors.num_colors;
}
uint64_t so_level_color_size( const so_level * level, uint64_t k ) {
	return level->level->colors.masks[ k ].size();
}
uint64_t so_level_color_nnz( const so_level * level, uint64_t k ) {
	return level->level->color_nnz[ k ];
}
void so_level_color_members( const so_level * level, uint64_t k, uint64_t * out ) {
	const auto members = level->level->colors.masks[ k ].members();
	std::memcpy( out, members.data(), members.size() * sizeof( uint64_t ) );
}
void so_level_csr( const so_level * level, uint64_t * row_offsets, uint64_t * cols, double * vals ) {
	const SparseMatrix & A = level->level->A;
	std::memcpy( row_offsets, A.row_offsets().data(), ( A.nrows() + 1 ) * sizeof( uint64_t ) );
	std::memcpy( cols, A.col_indices().data(), A.nnz() * sizeof( uint64_t ) );
	std::memcpy( vals, A.values().data(), A.nnz() * sizeof( double ) );
}
void so_level_diag( const so_level * level, double * out ) {
	vec_to( level->level->a_diag, out );
}
uint64_t so_level_nnz_visited( const so_level * level ) {
	return level->level->stats.nnz_visited;
}
void so_level_reset_stats( so_level * level ) {
	level->level->reset_stats();
}
int so_level_mxv( so_level * level, double * y, const double * x ) {
	if( y == x ) {
		return SO_INVALID_ARGUMENT;
	}
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector yv( n );
		mxv( yv, level->level->A, vec_from( x, n ) );
		vec_to( yv, y );
	} );
}

int so_rbgs_color_step( so_level * level, uint64_t k, double * z, const double * r ) {
	if( k >= level->level->colors.num_colors ) {
		return SO_INVALID_ARGUMENT;
	}
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		detail::rbgs_color_step( *level->level, k, zv, vec_from( r, n ) );
		vec_to( zv, z );
	} );
}

int so_rbgs_forward( so_level * level, double * z, const double * r ) {
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		rbgs_forward( *level->level, zv, vec_from( r, n ) );
		vec_to( zv, z );
	} );
}

int so_rbgs_backward( so_level * level, double * z, const double * r ) {
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		rbgs_backward( *level->level, zv, vec_from( r, n ) );
		vec_to( zv, z );
	} );
}

int so_rbgs_symmetric( so_level * level, double * z, const double * r, uint64_t sweeps ) {
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		rbgs_symmetric( *level->level, zv, vec_from( r, n ), SmootherConfig{ sweeps } );
		vec_to( zv, z );
	} );
}

int so_restrict_vector( so_level * level, const double * v_fine, double * out ) {
	return guarded( [ & ] {
		const DenseVector res = restrict_vector( *level->level, vec_from( v_fine, level->level->n() ) );
		vec_to( res, out );
	} );
}

int so_refine_and_add( so_level * level, double * z, const double * z_c ) {
	return guarded( [ & ] {
		if( !level->level->restriction ) {
			throw InvalidArgument( "no restriction" );
		}
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		refine_and_add( *level->level, zv, vec_from( z_c, level->level->restriction->nrows() ) );
		vec_to( zv, z );
	} );
}

int so_mg_vcycle( so_level * level, double * z, const double * r, uint64_t sweeps ) {
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		DenseVector zv = vec_from( z, n );
		mg_vcycle( *level->level, zv, vec_from( r, n ), SmootherConfig{ sweeps } );
		vec_to( zv, z );
	} );
}

int so_cg_solve( so_level * hierarchy, const double * b, const double * x0, const so_cg_config * cfg, double * x,
	double * history, uint64_t * iterations, int * converged ) {
	return guarded( [ & ] {
		const std::size_t n = hierarchy->level->n();
		CGConfig c;
		c.max_iters = cfg->max_iters;
		c.rtol = cfg->rtol;
		c.use_preconditioner = cfg->use_preconditioner != 0;
		if( cfg->has_fixed_iterations ) {
			c.fixed_iterations = cfg->fixed_iterations;
		}
		const CGResult res = cg_solve( *hierarchy->level, vec_from( b, n ), vec_from( x0, n ), c,
			SmootherConfig{ cfg->sweeps } );
		vec_to( res.solution, x );
		for( std::size_t k = 0; k < res.residual_history.size(); ++k ) {
			history[ k ] = res.residual_history[ k ];
		}
		*iterations = res.iterations;
		*converged = res.converged ? 1 : 0;
	} );
}

int so_residual_norm( so_level * level, const double * x, const double * b, double * out ) {
	return guarded( [ & ] {
		const std::size_t n = level->level->n();
		*out = residual_norm( level->level->A, vec_from( x, n ), vec_from( b, n ) );
	} );
}

} // extern "C"
