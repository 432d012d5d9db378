/*
 * slab_oracle.c — CPU oracle: a plain-C restatement of the reference's
 * arithmetic for the MG-preconditioned CG hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see slab_oracle.h). Never linked into, loaded by
 * or called from the product path.
 *
 * Parity status: PINNED against the reference headers themselves
 * (oracle/_ref/libslab_ref.so, built from /root/reference/proj/include by
 * oracle/Makefile) and against tests/golden/ (generated from those headers).
 *
 * Every function cites the reference file:line (relative to
 * /root/reference/proj/include/slab/) whose operation order it follows. The
 * contract that matters for bitwise parity:
 *   - no FMA contraction (reference CMakeLists.txt:8-14 has no -march): this
 *     file must be compiled with -ffp-contract=off;
 *   - row sums run over stored entries in ascending column order, product
 *     rounded, then added (operations.hpp:116-125);
 *   - dot sums 4096-element chunks left to right and combines the partials in
 *     chunk order (operations.hpp:61-91, parallel.hpp:70);
 *   - waxpby rounds both products, then adds (operations.hpp:103);
 *   - the smoother update is ((r - s) + z*d) / d (smoother.hpp:68).
 * OpenMP only splits independent iterations, so results do not depend on the
 * thread count (parallel.hpp:74-88).
 */
#include "slab_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define SO_REDUCTION_CHUNK 4096u /* parallel.hpp:70 */
#define SO_PARALLEL_GRAIN 2048u  /* parallel.hpp:67 */

static int so_thread_cap = 0;

const char * so_kind( void ) {
	return "port";
}

void so_set_threads( int threads ) { /* parallel.hpp:50 */
	so_thread_cap = threads;
}

int so_get_threads( void ) { /* parallel.hpp:55 */
#ifdef _OPENMP
	return so_thread_cap == 0 ? omp_get_max_threads() : so_thread_cap;
#else
	return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* problem generation                                                  */
/* ------------------------------------------------------------------ */

/* problem.hpp:80-82 */
uint64_t so_stencil_nnz( uint64_t nx, uint64_t ny, uint64_t nz ) {
	return ( 3 * nx - 2 ) * ( 3 * ny - 2 ) * ( 3 * nz - 2 );
}

/* problem.hpp:90-131: x-fastest ordering, neighbours ascending in (z,y,x),
 * 26.0 on the diagonal, -1.0 elsewhere. */
int so_build_stencil( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * row_offsets, uint64_t * cols, double * vals ) {
	if( nx < 2 || ny < 2 || nz < 2 ) {
		return SO_INVALID_ARGUMENT; /* problem.hpp:65-70 */
	}
	uint64_t at = 0;
	uint64_t row = 0;
	row_offsets[ 0 ] = 0;
	for( uint64_t iz = 0; iz < nz; ++iz ) {
		for( uint64_t iy = 0; iy < ny; ++iy ) {
			for( uint64_t ix = 0; ix < nx; ++ix ) {
				const uint64_t i = ix + nx * ( iy + ny * iz );
				for( uint64_t jz = iz > 0 ? iz - 1 : 0; jz < nz && jz <= iz + 1; ++jz ) {
					for( uint64_t jy = iy > 0 ? iy - 1 : 0; jy < ny && jy <= iy + 1; ++jy ) {
						for( uint64_t jx = ix > 0 ? ix - 1 : 0; jx < nx && jx <= ix + 1; ++jx ) {
							const uint64_t j = jx + nx * ( jy + ny * jz );
							cols[ at ] = j;
							vals[ at ] = j == i ? 26.0 : -1.0;
							++at;
						}
					}
				}
				row_offsets[ ++row ] = at;
			}
		}
	}
	return SO_OK;
}

/* problem.hpp:174-201: row c of R has its single 1.0 at fine (2cx,2cy,2cz). */
int so_build_restriction_cols( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t * cols ) {
	if( nx < 2 || ny < 2 || nz < 2 || nx % 2 || ny % 2 || nz % 2 ) {
		return SO_INVALID_ARGUMENT;
	}
	uint64_t c = 0;
	for( uint64_t cz = 0; cz < nz / 2; ++cz ) {
		for( uint64_t cy = 0; cy < ny / 2; ++cy ) {
			for( uint64_t cx = 0; cx < nx / 2; ++cx ) {
				cols[ c++ ] = 2 * cx + nx * ( 2 * cy + ny * 2 * cz );
			}
		}
	}
	return SO_OK;
}

/* ------------------------------------------------------------------ */
/* rng.hpp:35-65                                                       */
/* ------------------------------------------------------------------ */

uint64_t so_lcg_next( uint64_t state ) {
	return state * 6364136223846793005ULL + 1442695040888963407ULL;
}

uint64_t so_lcg_fill( uint64_t seed, double * out, uint64_t n ) {
	uint64_t state = seed;
	for( uint64_t i = 0; i < n; ++i ) {
		state = so_lcg_next( state );
		const double unit = (double) ( state >> 11 ) * 0x1.0p-53; /* rng.hpp:45-47 */
		out[ i ] = 2.0 * unit - 1.0;                               /* rng.hpp:50-52 */
	}
	return state;
}

/* ------------------------------------------------------------------ */
/* primitives                                                          */
/* ------------------------------------------------------------------ */

/* operations.hpp:61-91 */
double so_dot( const double * x, const double * y, uint64_t n ) {
	const uint64_t chunk = SO_REDUCTION_CHUNK;
	const uint64_t nchunks = ( n + chunk - 1 ) / chunk;
	if( nchunks <= 1 ) {
		double acc = 0.0;
		for( uint64_t i = 0; i < n; ++i ) {
			acc = acc + x[ i ] * y[ i ];
		}
		return acc;
	}
	double * partials = (double *) malloc( nchunks * sizeof( double ) );
	const int threads = so_get_threads();
	(void) threads;
	#pragma omp parallel for schedule( static ) num_threads( threads ) if( nchunks >= SO_PARALLEL_GRAIN )
	for( int64_t c = 0; c < (int64_t) nchunks; ++c ) {
		const uint64_t begin = (uint64_t) c * chunk;
		const uint64_t end = begin + chunk < n ? begin + chunk : n;
		double acc = 0.0;
		for( uint64_t i = begin; i < end; ++i ) {
			acc = acc + x[ i ] * y[ i ];
		}
		partials[ c ] = acc;
	}
	double acc = 0.0;
	for( uint64_t c = 0; c < nchunks; ++c ) {
		acc = acc + partials[ c ];
	}
	free( partials );
	return acc;
}

/* operations.hpp:97-106: two rounded products, one add; w may alias x or y */
void so_waxpby( double * w, double alpha, const double * x, double beta, const double * y, uint64_t n ) {
	const int threads = so_get_threads();
	(void) threads;
	#pragma omp parallel for schedule( static ) num_threads( threads ) if( n >= SO_PARALLEL_GRAIN )
	for( int64_t i = 0; i < (int64_t) n; ++i ) {
		w[ i ] = alpha * x[ i ] + beta * y[ i ];
	}
}

static void so_set_all( double * v, double value, uint64_t n ) { /* operations.hpp:49-54 */
	for( uint64_t i = 0; i < n; ++i ) {
		v[ i ] = value;
	}
}

/* operations.hpp:116-125 */
static inline double so_row_dot( const uint64_t * row_offsets, const uint64_t * cols, const double * vals, uint64_t row,
	const double * x ) {
	double acc = 0.0;
	for( uint64_t k = row_offsets[ row ]; k < row_offsets[ row + 1 ]; ++k ) {
		acc = acc + vals[ k ] * x[ cols[ k ] ];
	}
	return acc;
}

/* operations.hpp:164-167 */
void so_mxv_csr( double * y, uint64_t nrows, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	const double * x ) {
	const int threads = so_get_threads();
	(void) threads;
	#pragma omp parallel for schedule( static ) num_threads( threads ) if( nrows >= SO_PARALLEL_GRAIN )
	for( int64_t i = 0; i < (int64_t) nrows; ++i ) {
		y[ i ] = so_row_dot( row_offsets, cols, vals, (uint64_t) i, x );
	}
}

/* operations.hpp:168-174: only members are written */
void so_mxv_csr_masked( double * y, const uint64_t * members, uint64_t nmembers, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x ) {
	const int threads = so_get_threads();
	(void) threads;
	#pragma omp parallel for schedule( static ) num_threads( threads ) if( nmembers >= SO_PARALLEL_GRAIN )
	for( int64_t k = 0; k < (int64_t) nmembers; ++k ) {
		const uint64_t i = members[ k ];
		y[ i ] = so_row_dot( row_offsets, cols, vals, i, x );
	}
}

/* operations.hpp:180-188: serial scatter in row order */
void so_mxv_csr_transpose( double * y, uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets,
	const uint64_t * cols, const double * vals, const double * x ) {
	so_set_all( y, 0.0, ncols );
	for( uint64_t i = 0; i < nrows; ++i ) {
		for( uint64_t k = row_offsets[ i ]; k < row_offsets[ i + 1 ]; ++k ) {
			y[ cols[ k ] ] = y[ cols[ k ] ] + vals[ k ] * x[ i ];
		}
	}
}

/* operations.hpp:189-203 */
void so_mxv_csr_transpose_masked( double * y, const uint64_t * members, uint64_t nmembers, uint64_t nrows, uint64_t ncols,
	const uint64_t * row_offsets, const uint64_t * cols, const double * vals, const double * x ) {
	char * selected = (char *) calloc( ncols ? ncols : 1, 1 );
	for( uint64_t m = 0; m < nmembers; ++m ) {
		selected[ members[ m ] ] = 1;
		y[ members[ m ] ] = 0.0;
	}
	for( uint64_t i = 0; i < nrows; ++i ) {
		for( uint64_t k = row_offsets[ i ]; k < row_offsets[ i + 1 ]; ++k ) {
			if( selected[ cols[ k ] ] ) {
				y[ cols[ k ] ] = y[ cols[ k ] ] + vals[ k ] * x[ i ];
			}
		}
	}
	free( selected );
}

/* ------------------------------------------------------------------ */
/* levels                                                              */
/* ------------------------------------------------------------------ */

struct so_level {
	uint64_t dims[ 3 ];
	uint64_t n, nnz;
	uint64_t * row_offsets;
	uint64_t * cols;
	double * vals;
	double * a_diag;
	uint64_t num_colors;
	uint64_t * color_start; /* num_colors+1 offsets into members */
	uint64_t * members;     /* masks concatenated in color order, ascending inside a color */
	uint64_t * color_nnz;
	int has_restriction;
	uint64_t n_coarse;
	uint64_t * r_cols; /* restriction: one column per coarse row */
	struct so_level * coarser;
	double * s;
	double * f;
	double * r_c;
	double * z_c;
	uint64_t nnz_visited;
};

/* problem.hpp:143-166 */
static int so_extract_diagonal( so_level * L ) {
	L->a_diag = (double *) malloc( ( L->n ? L->n : 1 ) * sizeof( double ) );
	for( uint64_t i = 0; i < L->n; ++i ) {
		double value = 0.0;
		int found = 0;
		for( uint64_t k = L->row_offsets[ i ]; k < L->row_offsets[ i + 1 ]; ++k ) {
			if( L->cols[ k ] == i ) {
				value = L->vals[ k ];
				found = 1;
				break;
			}
		}
		if( !found || value == 0.0 ) {
			return SO_INVALID_ARGUMENT;
		}
		L->a_diag[ i ] = value;
	}
	return SO_OK;
}

/* coloring.hpp:114-158: greedy over pattern(A) united with pattern(A^T),
 * rows in increasing order, smallest colour not used by a coloured
 * neighbour. The neighbour visiting order is irrelevant, so the transpose
 * pattern is walked separately instead of being merged (coloring.hpp:61-102). */
static void so_greedy_color( so_level * L ) {
	const uint64_t n = L->n;
	const uint64_t unset = UINT64_MAX;
	/* pattern of A^T (sparse_matrix.hpp:178-200) */
	uint64_t * t_off = (uint64_t *) calloc( n + 2, sizeof( uint64_t ) );
	for( uint64_t k = 0; k < L->nnz; ++k ) {
		++t_off[ L->cols[ k ] + 1 ];
	}
	for( uint64_t i = 0; i < n; ++i ) {
		t_off[ i + 1 ] += t_off[ i ];
	}
	uint64_t * t_idx = (uint64_t *) malloc( ( L->nnz ? L->nnz : 1 ) * sizeof( uint64_t ) );
	uint64_t * cursor = (uint64_t *) malloc( ( n ? n : 1 ) * sizeof( uint64_t ) );
	memcpy( cursor, t_off, n * sizeof( uint64_t ) );
	for( uint64_t i = 0; i < n; ++i ) {
		for( uint64_t k = L->row_offsets[ i ]; k < L->row_offsets[ i + 1 ]; ++k ) {
			t_idx[ cursor[ L->cols[ k ] ]++ ] = i;
		}
	}
	uint64_t max_degree = 0;
	for( uint64_t i = 0; i < n; ++i ) {
		const uint64_t deg = ( L->row_offsets[ i + 1 ] - L->row_offsets[ i ] ) + ( t_off[ i + 1 ] - t_off[ i ] );
		if( deg > max_degree ) {
			max_degree = deg;
		}
	}
	uint64_t * color = (uint64_t *) malloc( ( n ? n : 1 ) * sizeof( uint64_t ) );
	for( uint64_t i = 0; i < n; ++i ) {
		color[ i ] = unset;
	}
	uint64_t * forbidden_at = (uint64_t *) malloc( ( max_degree + 2 ) * sizeof( uint64_t ) );
	for( uint64_t c = 0; c < max_degree + 2; ++c ) {
		forbidden_at[ c ] = unset;
	}
	uint64_t num_colors = 0;
	for( uint64_t i = 0; i < n; ++i ) {
		for( uint64_t k = L->row_offsets[ i ]; k < L->row_offsets[ i + 1 ]; ++k ) {
			const uint64_t j = L->cols[ k ];
			if( j != i && color[ j ] != unset ) {
				forbidden_at[ color[ j ] ] = i;
			}
		}
		for( uint64_t k = t_off[ i ]; k < t_off[ i + 1 ]; ++k ) {
			const uint64_t j = t_idx[ k ];
			if( j != i && color[ j ] != unset ) {
				forbidden_at[ color[ j ] ] = i;
			}
		}
		uint64_t chosen = 0;
		while( forbidden_at[ chosen ] == i ) {
			++chosen;
		}
		color[ i ] = chosen;
		if( chosen + 1 > num_colors ) {
			num_colors = chosen + 1;
		}
	}
	L->num_colors = num_colors;
	L->color_start = (uint64_t *) calloc( num_colors + 1, sizeof( uint64_t ) );
	for( uint64_t i = 0; i < n; ++i ) {
		++L->color_start[ color[ i ] + 1 ];
	}
	for( uint64_t c = 0; c < num_colors; ++c ) {
		L->color_start[ c + 1 ] += L->color_start[ c ];
	}
	L->members = (uint64_t *) malloc( ( n ? n : 1 ) * sizeof( uint64_t ) );
	uint64_t * fill = (uint64_t *) malloc( ( num_colors + 1 ) * sizeof( uint64_t ) );
	memcpy( fill, L->color_start, ( num_colors + 1 ) * sizeof( uint64_t ) );
	for( uint64_t i = 0; i < n; ++i ) {
		L->members[ fill[ color[ i ] ]++ ] = i; /* ascending i keeps members sorted */
	}
	/* problem.hpp:237-245 */
	L->color_nnz = (uint64_t *) calloc( num_colors + 1, sizeof( uint64_t ) );
	for( uint64_t c = 0; c < num_colors; ++c ) {
		for( uint64_t m = L->color_start[ c ]; m < L->color_start[ c + 1 ]; ++m ) {
			const uint64_t i = L->members[ m ];
			L->color_nnz[ c ] += L->row_offsets[ i + 1 ] - L->row_offsets[ i ];
		}
	}
	free( fill );
	free( forbidden_at );
	free( color );
	free( cursor );
	free( t_idx );
	free( t_off );
}

/* takes ownership of the three CSR arrays; problem.hpp:234-246 */
static int so_level_init( so_level * L, uint64_t n, uint64_t * row_offsets, uint64_t * cols, double * vals ) {
	memset( L, 0, sizeof( *L ) );
	L->dims[ 0 ] = n;
	L->dims[ 1 ] = 1;
	L->dims[ 2 ] = 1;
	L->n = n;
	L->nnz = row_offsets[ n ];
	L->row_offsets = row_offsets;
	L->cols = cols;
	L->vals = vals;
	const int rc = so_extract_diagonal( L );
	if( rc != SO_OK ) {
		return rc;
	}
	so_greedy_color( L );
	L->s = (double *) calloc( n ? n : 1, sizeof( double ) );
	L->f = (double *) calloc( n ? n : 1, sizeof( double ) );
	return SO_OK;
}

void so_level_destroy( so_level * L ) {
	while( L != NULL ) {
		so_level * next = L->coarser;
		free( L->row_offsets );
		free( L->cols );
		free( L->vals );
		free( L->a_diag );
		free( L->color_start );
		free( L->members );
		free( L->color_nnz );
		free( L->r_cols );
		free( L->s );
		free( L->f );
		free( L->r_c );
		free( L->z_c );
		free( L );
		L = next;
	}
}

/* sparse_matrix.hpp:96-124 */
static int so_validate_csr( uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets, const uint64_t * cols ) {
	if( row_offsets[ 0 ] != 0 ) {
		return SO_INVALID_ARGUMENT;
	}
	for( uint64_t i = 0; i < nrows; ++i ) {
		if( row_offsets[ i + 1 ] < row_offsets[ i ] ) {
			return SO_INVALID_ARGUMENT;
		}
		for( uint64_t k = row_offsets[ i ]; k < row_offsets[ i + 1 ]; ++k ) {
			if( cols[ k ] >= ncols ) {
				return SO_INVALID_ARGUMENT;
			}
			if( k > row_offsets[ i ] && cols[ k ] <= cols[ k - 1 ] ) {
				return SO_INVALID_ARGUMENT;
			}
		}
	}
	return SO_OK;
}

/* problem.hpp:253 (standalone level around an arbitrary square system) */
int so_level_from_csr( uint64_t n, const uint64_t * row_offsets, const uint64_t * cols, const double * vals,
	so_level ** out ) {
	*out = NULL;
	if( so_validate_csr( n, n, row_offsets, cols ) != SO_OK ) {
		return SO_INVALID_ARGUMENT;
	}
	const uint64_t nnz = row_offsets[ n ];
	uint64_t * ro = (uint64_t *) malloc( ( n + 1 ) * sizeof( uint64_t ) );
	uint64_t * co = (uint64_t *) malloc( ( nnz ? nnz : 1 ) * sizeof( uint64_t ) );
	double * va = (double *) malloc( ( nnz ? nnz : 1 ) * sizeof( double ) );
	memcpy( ro, row_offsets, ( n + 1 ) * sizeof( uint64_t ) );
	memcpy( co, cols, nnz * sizeof( uint64_t ) );
	memcpy( va, vals, nnz * sizeof( double ) );
	so_level * L = (so_level *) malloc( sizeof( so_level ) );
	const int rc = so_level_init( L, n, ro, co, va );
	if( rc != SO_OK ) {
		so_level_destroy( L );
		return rc;
	}
	*out = L;
	return SO_OK;
}

/* problem.hpp:284-319 */
int so_hierarchy_create( uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels, so_level ** out ) {
	*out = NULL;
	if( nx < 2 || ny < 2 || nz < 2 || levels < 1 || levels > 60 ) {
		return SO_INVALID_ARGUMENT;
	}
	const uint64_t divider = (uint64_t) 1 << ( levels - 1 );
	const uint64_t d[ 3 ] = { nx, ny, nz };
	for( int a = 0; a < 3; ++a ) {
		if( d[ a ] % divider != 0 || d[ a ] / divider < 2 ) {
			return SO_INVALID_ARGUMENT;
		}
	}
	so_level * head = NULL;
	so_level * tail = NULL;
	uint64_t lx = nx, ly = ny, lz = nz;
	for( uint64_t k = 0; k < levels; ++k ) {
		const uint64_t n = lx * ly * lz;
		const uint64_t nnz = so_stencil_nnz( lx, ly, lz );
		uint64_t * ro = (uint64_t *) malloc( ( n + 1 ) * sizeof( uint64_t ) );
		uint64_t * co = (uint64_t *) malloc( nnz * sizeof( uint64_t ) );
		double * va = (double *) malloc( nnz * sizeof( double ) );
		so_build_stencil( lx, ly, lz, ro, co, va );
		so_level * L = (so_level *) malloc( sizeof( so_level ) );
		const int rc = so_level_init( L, n, ro, co, va );
		if( rc != SO_OK ) {
			so_level_destroy( L );
			so_level_destroy( head );
			return rc;
		}
		L->dims[ 0 ] = lx;
		L->dims[ 1 ] = ly;
		L->dims[ 2 ] = lz;
		if( k + 1 < levels ) {
			L->has_restriction = 1;
			L->n_coarse = n / 8;
			L->r_cols = (uint64_t *) malloc( L->n_coarse * sizeof( uint64_t ) );
			so_build_restriction_cols( lx, ly, lz, L->r_cols );
			L->r_c = (double *) calloc( L->n_coarse, sizeof( double ) );
			L->z_c = (double *) calloc( L->n_coarse, sizeof( double ) );
			lx /= 2;
			ly /= 2;
			lz /= 2;
		}
		if( tail == NULL ) {
			head = L;
		} else {
			tail->coarser = L;
		}
		tail = L;
	}
	*out = head;
	return SO_OK;
}

so_level * so_level_coarser( so_level * L ) {
	return L->coarser;
}
uint64_t so_level_n( const so_level * L ) {
	return L->n;
}
uint64_t so_level_nnz( const so_level * L ) {
	return L->nnz;
}
void so_level_dims( const so_level * L, uint64_t dims[ 3 ] ) {
	memcpy( dims, L->dims, sizeof( L->dims ) );
}
uint64_t so_level_num_colors( const so_level * L ) {
	return L->num_colors;
}
uint64_t so_level_color_size( const so_level * L, uint64_t k ) {
	return L->color_start[ k + 1 ] - L->color_start[ k ];
}
uint64_t so_level_color_nnz( const so_level * L, uint64_t k ) {
	return L->color_nnz[ k ];
}
void so_level_color_members( const so_level * L, uint64_t k, uint64_t * out ) {
	memcpy( out, L->members + L->color_start[ k ], so_level_color_size( L, k ) * sizeof( uint64_t ) );
}
void so_level_csr( const so_level * L, uint64_t * row_offsets, uint64_t * cols, double * vals ) {
	memcpy( row_offsets, L->row_offsets, ( L->n + 1 ) * sizeof( uint64_t ) );
	memcpy( cols, L->cols, L->nnz * sizeof( uint64_t ) );
	memcpy( vals, L->vals, L->nnz * sizeof( double ) );
}
void so_level_diag( const so_level * L, double * out ) {
	memcpy( out, L->a_diag, L->n * sizeof( double ) );
}
uint64_t so_level_nnz_visited( const so_level * L ) {
	return L->nnz_visited;
}
void so_level_reset_stats( so_level * L ) { /* problem.hpp:271-276 */
	for( ; L != NULL; L = L->coarser ) {
		L->nnz_visited = 0;
	}
}
int so_level_mxv( so_level * L, double * y, const double * x ) {
	if( y == x ) {
		return SO_INVALID_ARGUMENT; /* operations.hpp:158-160 */
	}
	so_mxv_csr( y, L->n, L->row_offsets, L->cols, L->vals, x );
	return SO_OK;
}

/* ------------------------------------------------------------------ */
/* smoother.hpp                                                        */
/* ------------------------------------------------------------------ */

/* smoother.hpp:60-72: masked mxv into s, then the per-member update */
int so_rbgs_color_step( so_level * L, uint64_t k, double * z, const double * r ) {
	if( k >= L->num_colors ) {
		return SO_INVALID_ARGUMENT;
	}
	const uint64_t * members = L->members + L->color_start[ k ];
	const uint64_t count = L->color_start[ k + 1 ] - L->color_start[ k ];
	so_mxv_csr_masked( L->s, members, count, L->row_offsets, L->cols, L->vals, z );
	const double * s = L->s;
	const double * d = L->a_diag;
	const int threads = so_get_threads();
	(void) threads;
	#pragma omp parallel for schedule( static ) num_threads( threads ) if( count >= SO_PARALLEL_GRAIN )
	for( int64_t m = 0; m < (int64_t) count; ++m ) {
		const uint64_t i = members[ m ];
		z[ i ] = ( r[ i ] - s[ i ] + z[ i ] * d[ i ] ) / d[ i ];
	}
	L->nnz_visited += L->color_nnz[ k ];
	return SO_OK;
}

/* smoother.hpp:77-85 */
int so_rbgs_forward( so_level * L, double * z, const double * r ) {
	for( uint64_t k = 0; k < L->num_colors; ++k ) {
		so_rbgs_color_step( L, k, z, r );
	}
	return SO_OK;
}

/* smoother.hpp:92-100 */
int so_rbgs_backward( so_level * L, double * z, const double * r ) {
	for( uint64_t k = L->num_colors; k > 0; --k ) {
		so_rbgs_color_step( L, k - 1, z, r );
	}
	return SO_OK;
}

/* smoother.hpp:103-113 */
int so_rbgs_symmetric( so_level * L, double * z, const double * r, uint64_t sweeps ) {
	if( sweeps < 1 ) {
		return SO_INVALID_ARGUMENT;
	}
	for( uint64_t sweep = 0; sweep < sweeps; ++sweep ) {
		so_rbgs_forward( L, z, r );
		so_rbgs_backward( L, z, r );
	}
	return SO_OK;
}

/* ------------------------------------------------------------------ */
/* multigrid.hpp                                                       */
/* ------------------------------------------------------------------ */

/* multigrid.hpp:46-54: out = R v, a one-entry row sum 0 + 1.0*v[col] */
int so_restrict_vector( so_level * L, const double * v_fine, double * out ) {
	if( !L->has_restriction ) {
		return SO_INVALID_ARGUMENT;
	}
	for( uint64_t c = 0; c < L->n_coarse; ++c ) {
		double acc = 0.0;
		acc = acc + 1.0 * v_fine[ L->r_cols[ c ] ];
		out[ c ] = acc;
	}
	L->nnz_visited += L->n_coarse;
	return SO_OK;
}

/* multigrid.hpp:71-81: f = R^T z_c by serial scatter, then z = 1*z + 1*f */
int so_refine_and_add( so_level * L, double * z, const double * z_c ) {
	if( !L->has_restriction ) {
		return SO_INVALID_ARGUMENT;
	}
	so_set_all( L->f, 0.0, L->n );
	for( uint64_t c = 0; c < L->n_coarse; ++c ) {
		const uint64_t j = L->r_cols[ c ];
		L->f[ j ] = L->f[ j ] + 1.0 * z_c[ c ];
	}
	so_waxpby( z, 1.0, z, 1.0, L->f, L->n );
	L->nnz_visited += L->n_coarse;
	return SO_OK;
}

/* multigrid.hpp:87-116 */
int so_mg_vcycle( so_level * L, double * z, const double * r, uint64_t sweeps ) {
	int rc = so_rbgs_symmetric( L, z, r, sweeps );
	if( rc != SO_OK ) {
		return rc;
	}
	if( L->coarser == NULL ) {
		return SO_OK;
	}
	so_mxv_csr( L->f, L->n, L->row_offsets, L->cols, L->vals, z ); /* f <- A z */
	L->nnz_visited += L->nnz;
	so_waxpby( L->f, 1.0, r, -1.0, L->f, L->n ); /* f <- r - f */
	so_restrict_vector( L, L->f, L->r_c );
	so_set_all( L->z_c, 0.0, L->n_coarse );
	rc = so_mg_vcycle( L->coarser, L->z_c, L->r_c, sweeps );
	if( rc != SO_OK ) {
		return rc;
	}
	so_refine_and_add( L, z, L->z_c );
	return so_rbgs_symmetric( L, z, r, sweeps );
}

/* ------------------------------------------------------------------ */
/* cg.hpp                                                              */
/* ------------------------------------------------------------------ */

/* cg.hpp:59-67 */
int so_residual_norm( so_level * L, const double * x, const double * b, double * out ) {
	double * r = (double *) malloc( ( L->n ? L->n : 1 ) * sizeof( double ) );
	so_mxv_csr( r, L->n, L->row_offsets, L->cols, L->vals, x );
	so_waxpby( r, 1.0, b, -1.0, r, L->n );
	*out = sqrt( so_dot( r, r, L->n ) );
	free( r );
	return SO_OK;
}

/* cg.hpp:77-142 */
int so_cg_solve( so_level * H, const double * b, const double * x0, const so_cg_config * cfg, double * x,
	double * history, uint64_t * iterations, int * converged ) {
	if( !( cfg->rtol > 0.0 ) ) {
		return SO_INVALID_ARGUMENT;
	}
	if( cfg->max_iters < 1 ) {
		return SO_INVALID_ARGUMENT;
	}
	const uint64_t n = H->n;
	const uint64_t bytes = ( n ? n : 1 ) * sizeof( double );
	memcpy( x, x0, n * sizeof( double ) );
	double * r = (double *) calloc( 1, bytes );
	double * z = (double *) calloc( 1, bytes );
	double * p = (double *) calloc( 1, bytes );
	double * q = (double *) calloc( 1, bytes );
	int rc = SO_OK;

	so_mxv_csr( r, n, H->row_offsets, H->cols, H->vals, x );
	so_waxpby( r, 1.0, b, -1.0, r, n ); /* r = b - A x */

	const double b_norm = sqrt( so_dot( b, b, n ) );
	const double denom = b_norm > 0.0 ? b_norm : 1.0;
	double r_norm = sqrt( so_dot( r, r, n ) );
	uint64_t count = 0;
	history[ count++ ] = r_norm;

	const int fixed = cfg->has_fixed_iterations;
	const int already_converged = !fixed && r_norm / denom < cfg->rtol;
	const uint64_t limit = already_converged ? 0
		: fixed ? ( cfg->fixed_iterations < cfg->max_iters ? cfg->fixed_iterations : cfg->max_iters )
		: cfg->max_iters;

	double rho_prev = 0.0;
	for( uint64_t iter = 1; iter <= limit; ++iter ) {
		if( cfg->use_preconditioner ) {
			so_set_all( z, 0.0, n );
			rc = so_mg_vcycle( H, z, r, cfg->sweeps );
			if( rc != SO_OK ) {
				break;
			}
		} else {
			so_waxpby( z, 1.0, r, 0.0, r, n );
		}
		const double rho = so_dot( r, z, n );
		if( iter == 1 ) {
			so_waxpby( p, 1.0, z, 0.0, z, n );
		} else {
			so_waxpby( p, 1.0, z, rho / rho_prev, p, n );
		}
		so_mxv_csr( q, n, H->row_offsets, H->cols, H->vals, p );
		const double pq = so_dot( p, q, n );
		if( pq <= 0.0 ) {
			rc = SO_SOLVER_BREAKDOWN;
			break;
		}
		const double alpha = rho / pq;
		so_waxpby( x, 1.0, x, alpha, p, n );
		so_waxpby( r, 1.0, r, -alpha, q, n );
		rho_prev = rho;

		r_norm = sqrt( so_dot( r, r, n ) );
		history[ count++ ] = r_norm;
		if( !fixed && r_norm / denom < cfg->rtol ) {
			break;
		}
	}
	*iterations = count - 1;
	*converged = r_norm / denom < cfg->rtol;
	free( r );
	free( z );
	free( p );
	free( q );
	return rc;
}
