// containers.cu — context, vectors, matrices (SELL-32) and masks behind include/slab_b200.h.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.hpp"
#include "dist.hpp"
#include "kernels.cuh"

namespace slabgpu {

	void Sell::release() {
		if( slice_off ) cudaFree( slice_off );
		if( vals ) cudaFree( vals );
		if( cols ) cudaFree( cols );
		slice_off = nullptr;
		vals = nullptr;
		cols = nullptr;
		nrows = nslices = entries = 0;
		packed.release();
	}

	// ---------------------------------------------------------------- scratch

	void ensure_partials( slab_ctx_s * ctx, uint64_t count ) {
		if( count <= ctx->partials_cap ) {
			return;
		}
		// growing the scratch must not race with kernels still using the old one
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		if( ctx->d_partials ) {
			SLAB_CUDA( cudaFree( ctx->d_partials ) );
			ctx->d_partials = nullptr;
		}
		const uint64_t cap = std::max< uint64_t >( count, 1024 );
		SLAB_CUDA( cudaMalloc( &ctx->d_partials, cap * sizeof( double ) ) );
		ctx->partials_cap = cap;
		++ctx->scratch_gen; // graphs captured with the old pointer are stale (cg.cu, level.cu)
	}

	void ensure_pinned( slab_ctx_s * ctx, uint64_t doubles ) {
		if( doubles <= ctx->h_pinned_cap ) {
			return;
		}
		if( ctx->h_pinned ) {
			SLAB_CUDA( cudaFreeHost( ctx->h_pinned ) );
			ctx->h_pinned = nullptr;
		}
		const uint64_t cap = std::max< uint64_t >( doubles, 1024 );
		SLAB_CUDA( cudaMallocHost( &ctx->h_pinned, cap * sizeof( double ) ) );
		ctx->h_pinned_cap = cap;
	}

	double read_scalar( slab_ctx_s * ctx, int slot ) {
		ensure_pinned( ctx, 1 );
		SLAB_CUDA( cudaMemcpyAsync( ctx->h_pinned, ctx->d_scalars + slot, sizeof( double ), cudaMemcpyDeviceToHost,
			ctx->stream ) );
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		return ctx->h_pinned[ 0 ];
	}

	// ---------------------------------------------------------------- vectors

	slab_vec_s * vec_new( slab_ctx_s * ctx, uint64_t n, double value ) {
		std::unique_ptr< slab_vec_s > v( new slab_vec_s );
		v->ctx = ctx;
		v->n = n;
		// on a distributed context every vector carries room for the ghost points of the finest level
		v->n_alloc = n + ghost_capacity( ctx );
		SLAB_CUDA( cudaMalloc( &v->d, std::max< uint64_t >( v->n_alloc, 1 ) * sizeof( double ) ) );
		kern::fill( ctx->stream, v->d, n, value );
		if( v->n_alloc > n ) {
			kern::fill( ctx->stream, v->d + n, v->n_alloc - n, 0.0 );
		}
		return v.release();
	}

	void vec_free( slab_vec_s * v ) {
		delete v;
	}

	// ---------------------------------------------------------------- SELL builders

	namespace {

		// uploads slice widths -> offsets, allocates vals/cols. Returns the host offsets.
		std::vector< int64_t > sell_allocate( cudaStream_t st, Sell & S, int64_t nrows,
			const std::vector< int32_t > & widths ) {
			S.nrows = nrows;
			S.nslices = static_cast< int64_t >( widths.size() );
			std::vector< int64_t > off( widths.size() + 1, 0 );
			for( size_t s = 0; s < widths.size(); ++s ) {
				off[ s + 1 ] = off[ s ] + static_cast< int64_t >( widths[ s ] ) * kSlice;
			}
			S.entries = off.back();
			S.max_width = widths.empty() ? 0 : *std::max_element( widths.begin(), widths.end() );
			SLAB_CUDA( cudaMalloc( &S.slice_off, off.size() * sizeof( int64_t ) ) );
			SLAB_CUDA( cudaMalloc( &S.vals, std::max< int64_t >( S.entries, 1 ) * sizeof( double ) ) );
			SLAB_CUDA( cudaMalloc( &S.cols, std::max< int64_t >( S.entries, 1 ) * sizeof( int32_t ) ) );
			upload_sync( st, S.slice_off, off.data(), off.size() * sizeof( int64_t ) );
			return off;
		}

	} // namespace

	Sell sell_from_csr_rows( slab_ctx_s * ctx, const std::vector< int64_t > & rows, const uint64_t * ro,
		const uint64_t * co, const double * va ) {
		Sell S;
		const int64_t npos = static_cast< int64_t >( rows.size() );
		const int64_t nslices = ( npos + kSlice - 1 ) / kSlice;
		std::vector< int32_t > widths( nslices, 0 );
		for( int64_t p = 0; p < npos; ++p ) {
			if( rows[ p ] >= 0 ) {
				const int32_t len = static_cast< int32_t >( ro[ rows[ p ] + 1 ] - ro[ rows[ p ] ] );
				widths[ p / kSlice ] = std::max( widths[ p / kSlice ], len );
			}
		}
		try {
			const std::vector< int64_t > off = sell_allocate( ctx->stream, S, npos, widths );
			std::vector< double > vals( std::max< int64_t >( S.entries, 1 ), 0.0 );
			std::vector< int32_t > cols( std::max< int64_t >( S.entries, 1 ), -1 );
			for( int64_t p = 0; p < npos; ++p ) {
				if( rows[ p ] < 0 ) {
					continue;
				}
				const int64_t base = off[ p / kSlice ] + ( p % kSlice );
				const uint64_t begin = ro[ rows[ p ] ];
				const uint64_t end = ro[ rows[ p ] + 1 ];
				for( uint64_t k = begin; k < end; ++k ) {
					vals[ base + static_cast< int64_t >( k - begin ) * kSlice ] = va[ k ];
					cols[ base + static_cast< int64_t >( k - begin ) * kSlice ] = static_cast< int32_t >( co[ k ] );
				}
			}
			upload_sync( ctx->stream, S.vals, vals.data(), S.entries * sizeof( double ) );
			upload_sync( ctx->stream, S.cols, cols.data(), S.entries * sizeof( int32_t ) );
		} catch( ... ) {
			S.release();
			throw;
		}
		return S;
	}

	Decomp single_domain( uint64_t nx, uint64_t ny, uint64_t nz ) {
		return single_domain_decomp( static_cast< int >( nx ), static_cast< int >( ny ), static_cast< int >( nz ) );
	}

	Sell sell_stencil27( slab_ctx_s * ctx, const Decomp & D, const int32_t * d_rows, int64_t npos ) {
		Sell S;
		const int64_t nslices = ( npos + kSlice - 1 ) / kSlice;
		int32_t * d_widths = nullptr;
		try {
			SLAB_CUDA( cudaMalloc( &d_widths, std::max< int64_t >( nslices, 1 ) * sizeof( int32_t ) ) );
			kern::stencil_widths( ctx->stream, D, d_rows, npos, nslices, d_widths );
			std::vector< int32_t > widths( nslices );
			SLAB_CUDA( cudaMemcpyAsync( widths.data(), d_widths, nslices * sizeof( int32_t ), cudaMemcpyDeviceToHost,
				ctx->stream ) );
			SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
			sell_allocate( ctx->stream, S, npos, widths );
			kern::stencil_fill( ctx->stream, D, d_rows, npos, nslices, S.slice_off, S.vals, S.cols );
			SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		} catch( ... ) {
			if( d_widths ) cudaFree( d_widths );
			S.release();
			throw;
		}
		cudaFree( d_widths );
		return S;
	}

	// ---------------------------------------------------------------- matrices

	namespace {
		void check_dims( uint64_t nx, uint64_t ny, uint64_t nz ) { // problem.hpp:65-70
			if( nx < 2 || ny < 2 || nz < 2 ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "grid dimensions must all be at least 2, got " + std::to_string( nx ) + "x"
					+ std::to_string( ny ) + "x" + std::to_string( nz ) );
			}
			// (overflow-safe: a product that wraps around 2^64 must not slip under the limit)
			const uint64_t limit = uint64_t( 1 ) << 31;
			if( nx >= limit || ny >= limit || nz >= limit || nx > ( limit - 1 ) / ny || nx * ny > ( limit - 1 ) / nz ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "grid too large for 32-bit column indices on one device" );
			}
		}
	} // namespace

	slab_mat_s * mat_from_csr( slab_ctx_s * ctx, uint64_t nrows, uint64_t ncols, const uint64_t * ro,
		const uint64_t * co, const double * va, bool validate ) {
		if( validate ) { // sparse_matrix.hpp:96-124
			if( ro == nullptr || ro[ 0 ] != 0 ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "from_csr: row_offsets must have nrows+1 entries starting at 0" );
			}
			for( uint64_t i = 0; i < nrows; ++i ) {
				if( ro[ i + 1 ] < ro[ i ] ) {
					fail( SLAB_ERR_INVALID_ARGUMENT, "from_csr: row_offsets must be non-decreasing" );
				}
				for( uint64_t k = ro[ i ]; k < ro[ i + 1 ]; ++k ) {
					if( co[ k ] >= ncols ) {
						fail( SLAB_ERR_INVALID_ARGUMENT, "from_csr: column index out of range in row " + std::to_string( i ) );
					}
					if( k > ro[ i ] && co[ k ] <= co[ k - 1 ] ) {
						fail( SLAB_ERR_INVALID_ARGUMENT,
							"from_csr: columns must be strictly increasing in row " + std::to_string( i ) );
					}
				}
			}
		}
		if( nrows >= ( uint64_t( 1 ) << 31 ) || ncols >= ( uint64_t( 1 ) << 31 ) ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "matrix too large for 32-bit column indices on one device" );
		}
		std::unique_ptr< slab_mat_s > A( new slab_mat_s );
		A->ctx = ctx;
		A->nrows = nrows;
		A->ncols = ncols;
		A->nnz = ro[ nrows ];
		std::vector< int64_t > rows( nrows );
		std::iota( rows.begin(), rows.end(), int64_t( 0 ) );
		A->sell = sell_from_csr_rows( ctx, rows, ro, co, va );
		sell_pack( ctx, A->sell, nullptr );
		A->h_row_offsets.assign( ro, ro + nrows + 1 );
		A->h_cols.assign( co, co + A->nnz );
		A->h_vals.assign( va, va + A->nnz );
		A->has_host_csr = true;
		return A.release();
	}

	// natural-order rows as masks over the 27 offsets (tile.cu), verified against the coded copy; when the matrix
	// turns out regular, plane_spmv.cu computes its products without a matrix stream
	static void mat_box_tile( slab_ctx_s * ctx, slab_mat_s * A, const Decomp & D ) {
		if( ctx->dist != nullptr || D.n_ghost != 0 || !A->sell.packed.usable() || ( D.l[ 0 ] % 2 ) != 0 || !g_use_spmv_planes ) {
			return;
		}
		box_tile_build( ctx, A->sell, nullptr, D, A->tile );
		if( A->tile.usable() && A->tile.regular ) {
			kern::spmv_planes_prepare();
		} else {
			A->tile.release(); // the masks serve nothing else on a natural-order matrix
		}
	}

	slab_mat_s * mat_stencil27( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz ) {
		check_dims( nx, ny, nz );
		std::unique_ptr< slab_mat_s > A( new slab_mat_s );
		A->ctx = ctx;
		A->nrows = A->ncols = nx * ny * nz;
		A->nnz = ( 3 * nx - 2 ) * ( 3 * ny - 2 ) * ( 3 * nz - 2 ); // problem.hpp:80-82
		const Decomp D = single_domain( nx, ny, nz );
		A->sell = sell_stencil27( ctx, D, nullptr, static_cast< int64_t >( A->nrows ) );
		sell_pack( ctx, A->sell, nullptr );
		mat_box_tile( ctx, A.get(), D );
		return A.release();
	}

	// the rows a rank owns: n_local x n_local logical shape, columns >= n_local address ghost slots
	slab_mat_s * mat_stencil27_box( slab_ctx_s * ctx, const Decomp & D ) {
		for( int a = 0; a < 3; ++a ) {
			if( D.l[ a ] < 2 ) { // problem.hpp:65-70, per rank
				fail( SLAB_ERR_INVALID_ARGUMENT, "grid dimensions must all be at least 2" );
			}
		}
		if( static_cast< uint64_t >( D.n_local ) + static_cast< uint64_t >( D.n_ghost ) >= ( uint64_t( 1 ) << 31 ) ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "grid too large for 32-bit column indices on one device" );
		}
		std::unique_ptr< slab_mat_s > A( new slab_mat_s );
		A->ctx = ctx;
		A->nrows = A->ncols = static_cast< uint64_t >( D.n_local );
		uint64_t nnz = 1;
		for( int a = 0; a < 3; ++a ) {
			uint64_t sum = 0;
			for( int t = D.o[ a ]; t < D.o[ a ] + D.l[ a ]; ++t ) {
				sum += static_cast< uint64_t >( span_1d( t, D.g[ a ] ) );
			}
			nnz *= sum;
		}
		A->nnz = nnz; // equals (3nx-2)(3ny-2)(3nz-2) on a single domain (problem.hpp:80-82)
		A->sell = sell_stencil27( ctx, D, nullptr, static_cast< int64_t >( A->nrows ) );
		sell_pack( ctx, A->sell, nullptr, static_cast< int64_t >( A->ncols ) ); // columns >= ncols are ghost slots
		mat_box_tile( ctx, A.get(), D );
		return A.release();
	}

	slab_mat_s * mat_restriction( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz ) {
		check_dims( nx, ny, nz );
		if( nx % 2 || ny % 2 || nz % 2 ) { // problem.hpp:176-182
			fail( SLAB_ERR_INVALID_ARGUMENT, "build_restriction: every fine dimension must be even" );
		}
		std::unique_ptr< slab_mat_s > R( new slab_mat_s );
		R->ctx = ctx;
		R->nrows = ( nx / 2 ) * ( ny / 2 ) * ( nz / 2 );
		R->ncols = nx * ny * nz;
		R->nnz = R->nrows;
		const int64_t nslices = ( static_cast< int64_t >( R->nrows ) + kSlice - 1 ) / kSlice;
		std::vector< int32_t > widths( nslices, 1 );
		sell_allocate( ctx->stream, R->sell, static_cast< int64_t >( R->nrows ), widths );
		int32_t * d_fine = nullptr;
		SLAB_CUDA( cudaMalloc( &d_fine, std::max< uint64_t >( R->nrows, 1 ) * sizeof( int32_t ) ) );
		kern::injection_cols( ctx->stream, static_cast< int >( nx ), static_cast< int >( ny ), static_cast< int >( nz ),
			d_fine );
		kern::sell_single_entry( ctx->stream, d_fine, static_cast< int64_t >( R->nrows ), nslices, R->sell.vals,
			R->sell.cols );
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		cudaFree( d_fine );
		return R.release();
	}

	void mat_download_csr( slab_mat_s * A, uint64_t * ro, uint64_t * co, double * va ) {
		if( A->has_host_csr ) {
			std::memcpy( ro, A->h_row_offsets.data(), ( A->nrows + 1 ) * sizeof( uint64_t ) );
			std::memcpy( co, A->h_cols.data(), A->nnz * sizeof( uint64_t ) );
			std::memcpy( va, A->h_vals.data(), A->nnz * sizeof( double ) );
			return;
		}
		if( A->sell.plain_dropped() ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "the matrix was created with keep_plain = 0: only its coded copy is on the device, "
				"it cannot be downloaded or transposed" );
		}
		slab_ctx_s * ctx = A->ctx;
		const int64_t nrows = static_cast< int64_t >( A->nrows );
		int64_t * d_counts = nullptr;
		int64_t * d_off = nullptr;
		int64_t * d_cols = nullptr;
		double * d_vals = nullptr;
		try {
			SLAB_CUDA( cudaMalloc( &d_counts, std::max< int64_t >( nrows, 1 ) * sizeof( int64_t ) ) );
			kern::sell_row_counts( ctx->stream, A->sell.slice_off, A->sell.cols, nrows, d_counts );
			std::vector< int64_t > counts( nrows );
			SLAB_CUDA( cudaMemcpyAsync( counts.data(), d_counts, nrows * sizeof( int64_t ), cudaMemcpyDeviceToHost,
				ctx->stream ) );
			SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
			ro[ 0 ] = 0;
			for( int64_t i = 0; i < nrows; ++i ) {
				ro[ i + 1 ] = ro[ i ] + static_cast< uint64_t >( counts[ i ] );
			}
			if( ro[ nrows ] != A->nnz ) {
				fail( SLAB_ERR_INTERNAL, "download_csr: stored entry count disagrees with nnz" );
			}
			SLAB_CUDA( cudaMalloc( &d_off, ( nrows + 1 ) * sizeof( int64_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_cols, std::max< uint64_t >( A->nnz, 1 ) * sizeof( int64_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_vals, std::max< uint64_t >( A->nnz, 1 ) * sizeof( double ) ) );
			upload_sync( ctx->stream, d_off, ro, ( nrows + 1 ) * sizeof( int64_t ) );
			kern::sell_to_csr( ctx->stream, A->sell.slice_off, A->sell.vals, A->sell.cols, nrows, d_off, d_cols, d_vals );
			SLAB_CUDA( cudaMemcpyAsync( co, d_cols, A->nnz * sizeof( int64_t ), cudaMemcpyDeviceToHost, ctx->stream ) );
			SLAB_CUDA( cudaMemcpyAsync( va, d_vals, A->nnz * sizeof( double ), cudaMemcpyDeviceToHost, ctx->stream ) );
			SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		} catch( ... ) {
			cudaFree( d_counts );
			cudaFree( d_off );
			cudaFree( d_cols );
			cudaFree( d_vals );
			throw;
		}
		cudaFree( d_counts );
		cudaFree( d_off );
		cudaFree( d_cols );
		cudaFree( d_vals );
	}

	// Explicit transpose in SELL. The reference's transpose descriptor scatters A's rows serially in
	// row order (operations.hpp:180-188), so output j accumulates its contributions by ascending
	// row index starting from 0.0 — exactly an ordered row sum over row j of A^T with columns
	// ascending. Built once per matrix, on first use (setup cost, like sparse_matrix.hpp:178-200).
	slab_mat_s * mat_transposed( slab_mat_s * A ) {
		if( A->transposed ) {
			return A->transposed.get();
		}
		std::vector< uint64_t > ro( A->nrows + 1 ), co( std::max< uint64_t >( A->nnz, 1 ) );
		std::vector< double > va( std::max< uint64_t >( A->nnz, 1 ) );
		mat_download_csr( A, ro.data(), co.data(), va.data() );
		const uint64_t tn = A->ncols;
		std::vector< uint64_t > t_ro( tn + 1, 0 ), t_co( std::max< uint64_t >( A->nnz, 1 ) );
		std::vector< double > t_va( std::max< uint64_t >( A->nnz, 1 ) );
		for( uint64_t k = 0; k < A->nnz; ++k ) {
			++t_ro[ co[ k ] + 1 ];
		}
		for( uint64_t j = 0; j < tn; ++j ) {
			t_ro[ j + 1 ] += t_ro[ j ];
		}
		std::vector< uint64_t > cursor( t_ro.begin(), t_ro.end() - 1 );
		for( uint64_t i = 0; i < A->nrows; ++i ) {
			for( uint64_t k = ro[ i ]; k < ro[ i + 1 ]; ++k ) {
				const uint64_t at = cursor[ co[ k ] ]++;
				t_co[ at ] = i;
				t_va[ at ] = va[ k ];
			}
		}
		A->transposed.reset( mat_from_csr( A->ctx, tn, A->nrows, t_ro.data(), t_co.data(), t_va.data(), false ) );
		return A->transposed.get();
	}

	// ---------------------------------------------------------------- primitive ops

	void op_set_all( slab_vec_s * v, double value ) {
		// the ghost tail of a distributed vector mirrors the owners' values: a constant vector is
		// constant everywhere, so filling the tail too keeps the ghost copies consistent
		kern::fill( v->ctx->stream, v->d, v->n_alloc, value );
	}

	void op_waxpby( slab_vec_s * w, double alpha, slab_vec_s * x, double beta, slab_vec_s * y ) {
		if( w->n != x->n || x->n != y->n ) { // operations.hpp:99-101
			fail( SLAB_ERR_DIMENSION_MISMATCH, "waxpby: vector lengths differ" );
		}
		kern::waxpby( w->ctx->stream, w->d, alpha, x->d, beta, y->d, w->n );
	}

	void op_dot_to_slot( slab_vec_s * x, slab_vec_s * y, int slot, bool reduce ) {
		if( x->n != y->n ) { // operations.hpp:63-65
			fail( SLAB_ERR_DIMENSION_MISMATCH, "dot: vector lengths differ" );
		}
		slab_ctx_s * ctx = x->ctx;
		if( ctx->dot_mode == SLAB_DOT_EXACT ) {
			ensure_partials( ctx, ( x->n + kDotChunk - 1 ) / kDotChunk );
			kern::dot_exact( ctx->stream, x->d, y->d, x->n, ctx->d_partials, ctx->d_counter, ctx->d_scalars + slot );
		} else {
			ensure_partials( ctx, kern::dot_tree_blocks( x->n, ctx->sm_count ) );
			kern::dot_tree( ctx->stream, x->d, y->d, x->n, ctx->sm_count, ctx->d_partials, ctx->d_counter,
				ctx->d_scalars + slot );
		}
		if( reduce ) {
			allreduce_slot( ctx, slot ); // sum of the ranks' owned parts; no-op on one process
		}
	}

	double op_dot( slab_vec_s * x, slab_vec_s * y ) {
		op_dot_to_slot( x, y, S_TMP );
		return read_scalar( x->ctx, S_TMP );
	}

	void op_mxv( slab_vec_s * y, slab_mask_s * mask, slab_mat_s * A, slab_vec_s * x, unsigned desc ) {
		const bool transpose = ( desc & SLAB_DESC_TRANSPOSE ) != 0;
		const uint64_t out_len = transpose ? A->ncols : A->nrows; // operations.hpp:150-160
		const uint64_t in_len = transpose ? A->nrows : A->ncols;
		if( y->n != out_len || x->n != in_len ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "mxv: operand sizes do not match the matrix" );
		}
		if( mask != nullptr && mask->universe != out_len ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "mxv: mask universe differs from output length" );
		}
		if( y == x || y->d == x->d ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "mxv: output must not alias the input vector" );
		}
		slab_mat_s * M = transpose ? mat_transposed( A ) : A;
		cudaStream_t st = A->ctx->stream;
		if( A->plan != nullptr && !transpose ) {
			halo_exchange_plan( A->ctx, A->plan, x, -1 ); // ghost copies of x before the gather
		}
		if( mask == nullptr && !transpose && kern::spmv_planes_usable( M->tile, static_cast< int64_t >( M->nrows ), A->ctx->sm_count ) ) {
			kern::spmv_planes( st, A->ctx->sm_count, M->tile, x->d, y->d, nullptr, nullptr );
		} else if( mask == nullptr ) {
			kern::spmv( st, M->sell, x->d, y->d, static_cast< int64_t >( M->nrows ) );
		} else {
			kern::spmv_masked( st, M->sell, x->d, y->d, mask->d_members,
				static_cast< int64_t >( mask->count ) );
		}
	}

} // namespace slabgpu
