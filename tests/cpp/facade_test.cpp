// facade_test.cpp — the reference's own test shapes (proj/tests/test_multigrid.cpp:49-71,
// test_cg.cpp:155-175, test_smoother.cpp:134-155, test_algebra.cpp:216-224) written against the C++
// facade, i.e. the way a slab program reads after switching namespaces. Needs a B200.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "slab_b200.hpp"

namespace slab = slab_b200;
using namespace slab;

static int failures = 0;
#define CHECK( cond )                                                                  \
	do {                                                                               \
		if( !( cond ) ) {                                                              \
			std::printf( "FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond );                \
			++failures;                                                                \
		}                                                                              \
	} while( 0 )
#define CHECK_THROWS_AS( expr, type )                                                  \
	do {                                                                               \
		bool thrown = false;                                                           \
		try {                                                                          \
			expr;                                                                      \
		} catch( const type & ) {                                                      \
			thrown = true;                                                             \
		} catch( ... ) {                                                               \
		}                                                                              \
		if( !thrown ) {                                                                \
			std::printf( "FAIL %s:%d  %s did not throw %s\n", __FILE__, __LINE__, #expr, #type ); \
			++failures;                                                                \
		}                                                                              \
	} while( 0 )

int main() {
	Context ctx( 0 );

	{ // one cycle equals its scripted composition (test_multigrid.cpp:49-71)
		ProblemLevel direct = build_hierarchy( ctx, { 8, 8, 8 }, 2 );
		ProblemLevel scripted = build_hierarchy( ctx, { 8, 8, 8 }, 2 );
		Lcg64 rng( 7 );
		const DenseVector r = random_vector( ctx, direct.n(), rng );
		DenseVector z( ctx, direct.n(), 0.0 );
		mg_vcycle( direct, z, r );

		DenseVector w( ctx, scripted.n(), 0.0 );
		rbgs_symmetric( scripted, w, r );
		DenseVector f( ctx, scripted.n() );
		const SparseMatrix A = scripted.A();
		mxv( f, A, w );
		waxpby( f, 1.0, r, -1.0, f );
		ProblemLevel coarse = scripted.coarser();
		DenseVector r_c( ctx, coarse.n() );
		restrict_vector( scripted, f, r_c );
		DenseVector z_c( ctx, coarse.n(), 0.0 );
		rbgs_symmetric( coarse, z_c, r_c );
		refine_and_add( scripted, w, z_c );
		rbgs_symmetric( scripted, w, r );
		CHECK( z == w );
	}

	{ // fixed-iteration runs repeat bit-identically (test_cg.cpp:155-165) and the 16^3 golden head
		ProblemLevel h = build_hierarchy( ctx, { 16, 16, 16 }, 4 );
		const DenseVector ones( ctx, h.n(), 1.0 );
		DenseVector b( ctx, h.n() );
		const SparseMatrix A = h.A();
		mxv( b, A, ones );
		const DenseVector x0( ctx, h.n(), 0.0 );
		CGConfig cfg;
		cfg.max_iters = 50;
		cfg.fixed_iterations = 50;
		const CGResult first = cg_solve( ctx, h, b, x0, cfg );
		const CGResult second = cg_solve( ctx, h, b, x0, cfg );
		CHECK( first.iterations == 50 );
		CHECK( first.residual_history == second.residual_history );
		CHECK( first.solution == second.solution );
		// BASELINE.md §4, generated from the reference headers
		CHECK( first.residual_history[ 0 ] == 368.7058448139926 );
		CHECK( first.residual_history[ 1 ] == 89.569064584234326 );
		CHECK( first.residual_history[ 16 ] == 1.6520315629824046e-08 );
		CHECK( first.residual_history[ 50 ] == 2.9213507058910168e-33 );
		CHECK( std::abs( residual_norm( A, first.solution, b ) ) <= 1e-10 * std::sqrt( dot( b, b ) ) );
	}

	{ // symmetric = forward then backward; argument validation (test_smoother.cpp:134-155)
		ProblemLevel level = build_hierarchy( ctx, { 2, 2, 4 }, 1 );
		Lcg64 rng( 17 );
		const DenseVector r = random_vector( ctx, level.n(), rng );
		DenseVector composed( ctx, level.n(), 0.0 );
		rbgs_forward( level, composed, r );
		rbgs_backward( level, composed, r );
		DenseVector direct( ctx, level.n(), 0.0 );
		rbgs_symmetric( level, direct, r );
		CHECK( direct == composed );
		CHECK( level.stats().nnz_visited == 4 * level.A().nnz() );
		// the 27-point operator repeats at most 27 (offset, value) pairs: both copies are dictionary-coded
		CHECK( level.format_info().packed == 1 && level.format_info().escaped_rows == 0 );
		CHECK( level.A().format_info().packed == 1 && level.A().format_info().dict_size >= 2 && level.A().format_info().dict_size <= 28 );
		CHECK_THROWS_AS( rbgs_symmetric( level, direct, r, SmootherConfig{ 0 } ), InvalidArgument );
		DenseVector wrong( ctx, 3 );
		CHECK_THROWS_AS( rbgs_forward( level, wrong, r ), DimensionMismatch );
	}

	{ // mxv rejects shape mismatch and aliasing (test_algebra.cpp:216-224); breakdown (test_cg.cpp:177-182)
		const SparseMatrix A = build_matrix( ctx, { 2, 2, 2 } );
		DenseVector x( ctx, 8, 1.0 ), y7( ctx, 7 );
		CHECK_THROWS_AS( mxv( y7, A, x ), DimensionMismatch );
		CHECK_THROWS_AS( mxv( x, A, x ), InvalidArgument );
		CHECK_THROWS_AS( build_hierarchy( ctx, { 6, 4, 4 }, 3 ), InvalidArgument );
		ProblemLevel neg( ctx, 3, { 0, 1, 2, 3 }, { 0, 1, 2 }, { -1.0, -1.0, -1.0 } );
		const DenseVector b( ctx, 3, 1.0 ), x0( ctx, 3, 0.0 );
		CGConfig plain;
		plain.use_preconditioner = false;
		CHECK_THROWS_AS( cg_solve( ctx, neg, b, x0, plain ), SolverBreakdown );
	}

	{ // symmetry test passes on a generated hierarchy (test_bench.cpp:55-62)
		ProblemLevel hierarchy = build_hierarchy( ctx, { 8, 8, 8 }, 3 );
		const SymmetryReport verdict = symmetry_test( ctx, hierarchy, 123 );
		CHECK( verdict.matrix_pass );
		CHECK( verdict.precond_pass );
		CHECK( verdict.tolerance > 0.0 );
		CHECK( !verdict.skipped );
	}

	std::printf( failures == 0 ? "facade_test: all checks passed\n" : "facade_test: %d failure(s)\n", failures );
	return failures == 0 ? 0 : 1;
}
