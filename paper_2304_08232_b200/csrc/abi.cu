// abi.cu — the extern "C" surface declared in include/slab_b200.h. Every entry point
// translates internal exceptions into status codes; argument checks precede any work.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "common.hpp"
#include "dist.hpp"
#include "kernels.cuh"

using namespace slabgpu;

namespace {

	thread_local std::string t_last_error;

	template< class F >
	int guarded( F && f ) {
		try {
			f();
			return SLAB_OK;
		} catch( const Error & e ) {
			t_last_error = e.message;
			return e.status;
		} catch( const std::bad_alloc & ) {
			t_last_error = "host allocation failed";
			return SLAB_ERR_INTERNAL;
		} catch( const std::exception & e ) {
			t_last_error = e.what();
			return SLAB_ERR_INTERNAL;
		}
	}

	void need( const void * p, const char * what ) {
		if( p == nullptr ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, std::string( what ) + ": null handle or pointer" );
		}
	}

	void same_ctx( const slab_ctx_s * a, const slab_ctx_s * b ) {
		if( a != b ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "operands belong to different contexts" );
		}
	}

	void bind( slab_ctx_s * ctx ) {
		SLAB_CUDA( cudaSetDevice( ctx->device ) );
	}

} // namespace

extern "C" {

int slab_abi_version( void ) {
	return SLAB_B200_ABI_VERSION;
}

const char * slab_last_error( void ) {
	return t_last_error.c_str();
}

const char * slab_status_name( int status ) {
	switch( status ) {
		case SLAB_OK: return "ok";
		case SLAB_ERR_DIMENSION_MISMATCH: return "DimensionMismatch";
		case SLAB_ERR_INVALID_ARGUMENT: return "InvalidArgument";
		case SLAB_ERR_SOLVER_BREAKDOWN: return "SolverBreakdown";
		case SLAB_ERR_CUDA: return "CudaError";
		default: return "InternalError";
	}
}

int slab_set_programmatic_launch( int enabled ) {
	g_use_pdl = enabled ? 1 : 0;
	return SLAB_OK;
}

int slab_set_tuning( const char * key, int64_t value ) {
	return guarded( [ & ] {
		need( key, "slab_set_tuning" );
		const std::string k( key );
		if( k == "stream_rows" ) {
			g_stream_rows = value;
		} else if( k == "stream_variant" ) {
			g_stream_variant = static_cast< int >( value );
		} else if( k == "pdl" ) {
			g_use_pdl = value ? 1 : 0;
		} else if( k == "packed" ) {
			g_use_packed = value ? 1 : 0;
		} else if( k == "pack_build" ) {
			g_pack_build = value ? 1 : 0;
		} else if( k == "keep_plain" ) {
			g_keep_plain = value ? 1 : 0;
		} else if( k == "packed_block" ) {
			g_packed_block = static_cast< int >( value );
		} else if( k == "packed_rows" ) {
			g_packed_rows = static_cast< int >( value );
		} else if( k == "packed_rows_spmv" ) {
			g_packed_rows_spmv = static_cast< int >( value );
		} else if( k == "packed_multi_min_rows" ) {
			g_packed_multi_min_rows = value;
		} else if( k == "cluster_rows" ) {
			g_cluster_rows = value;
		} else if( k == "packed_batch" ) {
			g_packed_batch = static_cast< int >( value );
		} else if( k == "packed_min_rows" ) {
			g_packed_min_rows = value;
		} else if( k == "tile" ) {
			g_use_tile = value ? 1 : 0;
		} else if( k == "tile_min_rows" ) {
			g_tile_min_rows = value;
		} else if( k == "tile_ty" ) {
			g_tile_ty = static_cast< int >( value );
		} else if( k == "tile_cz" ) {
			g_tile_cz = static_cast< int >( value );
		} else if( k == "tile_ns" ) {
			g_tile_ns = static_cast< int >( value );
		} else if( k == "planes" ) {
			g_use_planes = value ? 1 : 0;
		} else if( k == "dot_tile" ) {
			g_dot_tile = static_cast< int >( value );
		} else if( k == "dot_cpb" ) {
			g_dot_cpb = static_cast< int >( value );
		} else if( k == "plane_autotune" ) {
			g_plane_autotune = value ? 1 : 0;
		} else if( k == "lazy_x" ) {
			g_lazy_x = static_cast< int >( value ); // 0 off, 1 for systems of at least 2^20 rows, 2 always
		} else if( k == "lazy_x_prio" ) {
			g_lazy_x_prio = value ? 1 : 0;
		} else if( k == "inline_record" ) {
			g_inline_record = value ? 1 : 0;
		} else if( k == "iter_batch" ) {
			g_iter_batch = static_cast< int >( value );
		} else if( k == "lazy_x_blocks" ) {
			g_lazy_x_blocks = static_cast< int >( value );
		} else if( k == "side_rr" ) {
			g_side_rr = value ? 1 : 0;
		} else if( k == "fuse_rz" ) {
			g_fuse_rz = static_cast< int >( value ); // 0 off, 1 for systems of at least 2^19 rows, 2 always
		} else if( k == "plane_pad_lines" ) {
			g_plane_pad_lines = static_cast< int >( value );
		} else if( k == "plane_warp_sync" ) {
			g_plane_warp_sync = value ? 1 : 0;
		} else if( k == "spmv_planes" ) {
			g_use_spmv_planes = value ? 1 : 0;
		} else if( k == "spmv_plane_min_rows" ) {
			g_spmv_plane_min_rows = value;
		} else if( k == "spmv_plane_ty" ) {
			g_spmv_plane_ty = static_cast< int >( value );
		} else if( k == "spmv_plane_cz" ) {
			g_spmv_plane_cz = static_cast< int >( value );
		} else if( k == "spmv_plane_ns" ) {
			g_spmv_plane_ns = static_cast< int >( value );
		} else if( k == "plane_min_rows" ) {
			g_plane_min_rows = value;
		} else if( k == "plane_ty" ) {
			g_plane_ty = static_cast< int >( value );
		} else if( k == "plane_cz" ) {
			g_plane_cz = static_cast< int >( value );
		} else if( k == "plane_ns" ) {
			g_plane_ns = static_cast< int >( value );
		} else if( k == "plane_rows" ) {
			g_plane_rows = static_cast< int >( value );
		} else if( k == "plane_unit" ) {
			g_plane_unit = value ? 1 : 0;
		} else if( k == "halo_overlap" ) {
			g_halo_overlap = value ? 1 : 0;
		} else if( k == "l2_window" ) {
			g_l2_window = static_cast< int >( value );
		} else {
			fail( SLAB_ERR_INVALID_ARGUMENT, "slab_set_tuning: unknown key " + k );
		}
		++g_tuning_epoch;
	} );
}

uint64_t slab_launch_count( void ) {
	return g_launch_count;
}

// ---------------------------------------------------------------- context

int slab_ctx_create( int device, slab_ctx_t * out ) {
	return guarded( [ & ] {
		need( out, "slab_ctx_create" );
		*out = nullptr;
		int count = 0;
		const cudaError_t err = cudaGetDeviceCount( &count );
		if( err != cudaSuccess || count == 0 ) {
			fail( SLAB_ERR_CUDA, std::string( "no CUDA device available (there is no CPU fallback): " )
				+ cudaGetErrorString( err ) );
		}
		if( device < 0 || device >= count ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "device index out of range" );
		}
		SLAB_CUDA( cudaSetDevice( device ) );
		cudaDeviceProp prop{};
		SLAB_CUDA( cudaGetDeviceProperties( &prop, device ) );
		if( prop.major < 10 ) {
			fail( SLAB_ERR_CUDA, std::string( "device " ) + prop.name + " is sm_" + std::to_string( prop.major )
				+ std::to_string( prop.minor ) + "; this library is built for sm_100a only" );
		}
		// performance knobs from the environment (never change results; see slab_set_tuning)
		if( const char * v = std::getenv( "SLAB_PDL" ) ) {
			g_use_pdl = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_STREAM_ROWS" ) ) {
			g_stream_rows = std::atoll( v );
		}
		if( const char * v = std::getenv( "SLAB_STREAM_VARIANT" ) ) {
			g_stream_variant = std::atoi( v );
		}
		if( const char * v = std::getenv( "SLAB_TILE" ) ) {
			g_use_tile = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_PACKED" ) ) {
			g_use_packed = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_CLUSTER_ROWS" ) ) {
			g_cluster_rows = std::atoll( v );
		}
		if( const char * v = std::getenv( "SLAB_KEEP_PLAIN" ) ) {
			g_keep_plain = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_PACK_BUILD" ) ) {
			g_pack_build = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_PACKED_BLOCK" ) ) {
			g_packed_block = std::atoi( v );
		}
		if( const char * v = std::getenv( "SLAB_HALO_OVERLAP" ) ) {
			g_halo_overlap = std::atoi( v ) ? 1 : 0;
		}
		if( const char * v = std::getenv( "SLAB_L2_WINDOW" ) ) {
			g_l2_window = std::atoi( v );
		}
		// L2 persisting carve-out for the vector that fine-level colour steps re-gather (kernels.cu)
		if( prop.persistingL2CacheMaxSize > 0 && g_l2_window ) {
			if( cudaDeviceSetLimit( cudaLimitPersistingL2CacheSize, static_cast< size_t >( prop.persistingL2CacheMaxSize ) )
				== cudaSuccess ) {
				g_l2_persist_bytes = static_cast< size_t >( prop.persistingL2CacheMaxSize );
				g_l2_window_max = static_cast< size_t >( prop.accessPolicyMaxWindowSize );
			} else {
				cudaGetLastError();
			}
		}
		std::unique_ptr< slab_ctx_s > ctx( new slab_ctx_s );
		ctx->device = device;
		ctx->sm_count = prop.multiProcessorCount;
		ctx->cc_major = prop.major;
		ctx->cc_minor = prop.minor;
		ctx->hbm_bytes = prop.totalGlobalMem;
		{
			int least = 0, greatest = 0; // the main stream above the lazy-x stream (created below with the least priority)
			SLAB_CUDA( cudaDeviceGetStreamPriorityRange( &least, &greatest ) );
			SLAB_CUDA( cudaStreamCreateWithPriority( &ctx->stream, cudaStreamNonBlocking, greatest ) );
		}
		kern::dot_exact_prepare();
		SLAB_CUDA( cudaMalloc( &ctx->d_scalars, S_COUNT * sizeof( double ) ) );
		SLAB_CUDA( cudaMemset( ctx->d_scalars, 0, S_COUNT * sizeof( double ) ) );
		SLAB_CUDA( cudaMalloc( &ctx->d_counter, 2 * sizeof( unsigned int ) ) );
		SLAB_CUDA( cudaMemset( ctx->d_counter, 0, 2 * sizeof( unsigned int ) ) );
		SLAB_CUDA( cudaStreamCreateWithFlags( &ctx->side_stream, cudaStreamNonBlocking ) );
		SLAB_CUDA( cudaEventCreateWithFlags( &ctx->side_fork, cudaEventDisableTiming ) );
		SLAB_CUDA( cudaEventCreateWithFlags( &ctx->side_join, cudaEventDisableTiming ) );
		{
			int least = 0, greatest = 0;
			SLAB_CUDA( cudaDeviceGetStreamPriorityRange( &least, &greatest ) );
			SLAB_CUDA( cudaStreamCreateWithPriority( &ctx->lazy_stream, cudaStreamNonBlocking, least ) );
		}
		SLAB_CUDA( cudaEventCreateWithFlags( &ctx->lazy_fork, cudaEventDisableTiming ) );
		SLAB_CUDA( cudaEventCreateWithFlags( &ctx->lazy_join, cudaEventDisableTiming ) );
		SLAB_CUDA( cudaDeviceSynchronize() ); // the memsets ran on the legacy stream
		SLAB_CUDA( cudaEventCreate( &ctx->timer_start ) );
		SLAB_CUDA( cudaEventCreate( &ctx->timer_stop ) );
		SLAB_CUDA( cudaEventCreate( &ctx->solve_start ) );
		SLAB_CUDA( cudaEventCreate( &ctx->solve_stop ) );
		ensure_partials( ctx.get(), 4096 );
		ensure_pinned( ctx.get(), 1024 );
		*out = ctx.release();
	} );
}

int slab_ctx_destroy( slab_ctx_t ctx ) {
	return guarded( [ & ] {
		if( ctx == nullptr ) {
			return;
		}
		cudaSetDevice( ctx->device );
		cudaStreamSynchronize( ctx->stream );
		dist_destroy( ctx );
		spans_discard( ctx );
		for( cudaEvent_t e : ctx->event_pool ) {
			cudaEventDestroy( e );
		}
		cudaFree( ctx->d_scalars );
		cudaFree( ctx->d_partials );
		cudaFree( ctx->d_counter );
		if( ctx->h_pinned ) cudaFreeHost( ctx->h_pinned );
		cudaEventDestroy( ctx->timer_start );
		cudaEventDestroy( ctx->timer_stop );
		cudaEventDestroy( ctx->solve_start );
		cudaEventDestroy( ctx->solve_stop );
		cudaFree( ctx->d_partials_side );
		cudaEventDestroy( ctx->side_fork );
		cudaEventDestroy( ctx->side_join );
		cudaStreamDestroy( ctx->side_stream );
		cudaEventDestroy( ctx->lazy_fork );
		cudaEventDestroy( ctx->lazy_join );
		cudaStreamDestroy( ctx->lazy_stream );
		cudaStreamDestroy( ctx->stream );
		delete ctx;
	} );
}

int slab_ctx_sync( slab_ctx_t ctx ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_sync" );
		bind( ctx );
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
	} );
}

int slab_ctx_set_dot_mode( slab_ctx_t ctx, int mode ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_set_dot_mode" );
		if( mode != SLAB_DOT_EXACT && mode != SLAB_DOT_TREE ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "unknown dot mode" );
		}
		ctx->dot_mode = mode;
	} );
}

int slab_ctx_get_dot_mode( slab_ctx_t ctx, int * mode ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_get_dot_mode" );
		need( mode, "slab_ctx_get_dot_mode" );
		*mode = ctx->dot_mode;
	} );
}

int slab_ctx_set_graphs( slab_ctx_t ctx, int enabled ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_set_graphs" );
		ctx->use_graphs = enabled ? 1 : 0;
	} );
}

int slab_ctx_set_profiling( slab_ctx_t ctx, int enabled ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_set_profiling" );
		bind( ctx );
		spans_resolve( ctx );
		ctx->profiling = enabled ? 1 : 0;
	} );
}

int slab_ctx_set_fused_transfers( slab_ctx_t ctx, int enabled ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_set_fused_transfers" );
		ctx->fused_transfers = enabled ? 1 : 0;
	} );
}

int slab_ctx_timer_start( slab_ctx_t ctx ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_timer_start" );
		bind( ctx );
		SLAB_CUDA( cudaEventRecord( ctx->timer_start, ctx->stream ) );
	} );
}

int slab_ctx_timer_stop( slab_ctx_t ctx, double * elapsed_ms ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_timer_stop" );
		need( elapsed_ms, "slab_ctx_timer_stop" );
		bind( ctx );
		SLAB_CUDA( cudaEventRecord( ctx->timer_stop, ctx->stream ) );
		SLAB_CUDA( cudaEventSynchronize( ctx->timer_stop ) );
		float ms = 0.0f;
		SLAB_CUDA( cudaEventElapsedTime( &ms, ctx->timer_start, ctx->timer_stop ) );
		*elapsed_ms = ms;
	} );
}

int slab_ctx_device_info( slab_ctx_t ctx, int * sm_count, int * cc_major, int * cc_minor, uint64_t * hbm_bytes ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_device_info" );
		if( sm_count ) *sm_count = ctx->sm_count;
		if( cc_major ) *cc_major = ctx->cc_major;
		if( cc_minor ) *cc_minor = ctx->cc_minor;
		if( hbm_bytes ) *hbm_bytes = ctx->hbm_bytes;
	} );
}

// ---------------------------------------------------------------- vectors

int slab_vec_create( slab_ctx_t ctx, uint64_t n, double value, slab_vec_t * out ) {
	return guarded( [ & ] {
		need( ctx, "slab_vec_create" );
		need( out, "slab_vec_create" );
		*out = nullptr;
		bind( ctx );
		*out = vec_new( ctx, n, value );
	} );
}

int slab_vec_destroy( slab_vec_t v ) {
	return guarded( [ & ] {
		if( v ) {
			cudaSetDevice( v->ctx->device );
			cudaStreamSynchronize( v->ctx->stream );
			vec_free( v );
		}
	} );
}

int slab_vec_size( slab_vec_t v, uint64_t * n ) {
	return guarded( [ & ] {
		need( v, "slab_vec_size" );
		need( n, "slab_vec_size" );
		*n = v->n;
	} );
}

int slab_vec_upload( slab_vec_t v, const double * host, uint64_t n ) {
	return guarded( [ & ] {
		need( v, "slab_vec_upload" );
		if( n != v->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "upload: host length differs from the vector length" );
		}
		if( n == 0 ) {
			return;
		}
		need( host, "slab_vec_upload" );
		bind( v->ctx );
		SLAB_CUDA( cudaMemcpyAsync( v->d, host, n * sizeof( double ), cudaMemcpyHostToDevice, v->ctx->stream ) );
		SLAB_CUDA( cudaStreamSynchronize( v->ctx->stream ) );
	} );
}

int slab_vec_download( slab_vec_t v, double * host, uint64_t n ) {
	return guarded( [ & ] {
		need( v, "slab_vec_download" );
		if( n != v->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "download: host length differs from the vector length" );
		}
		if( n == 0 ) {
			return;
		}
		need( host, "slab_vec_download" );
		bind( v->ctx );
		SLAB_CUDA( cudaMemcpyAsync( host, v->d, n * sizeof( double ), cudaMemcpyDeviceToHost, v->ctx->stream ) );
		SLAB_CUDA( cudaStreamSynchronize( v->ctx->stream ) );
	} );
}

int slab_vec_copy( slab_vec_t dst, slab_vec_t src ) {
	return guarded( [ & ] {
		need( dst, "slab_vec_copy" );
		need( src, "slab_vec_copy" );
		same_ctx( dst->ctx, src->ctx );
		if( dst->n != src->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "copy: vector lengths differ" );
		}
		bind( dst->ctx );
		if( dst->d != src->d && dst->n > 0 ) {
			SLAB_CUDA( cudaMemcpyAsync( dst->d, src->d, dst->n * sizeof( double ), cudaMemcpyDeviceToDevice,
				dst->ctx->stream ) );
		}
	} );
}

// rng.hpp:35-65 — the sequence is inherently serial, so it is generated on the host and uploaded
int slab_vec_fill_lcg( slab_vec_t v, uint64_t seed, uint64_t * state_out ) {
	return guarded( [ & ] {
		need( v, "slab_vec_fill_lcg" );
		bind( v->ctx );
		std::vector< double > host( v->n );
		uint64_t state = seed;
		for( uint64_t i = 0; i < v->n; ++i ) {
			state = state * 6364136223846793005ULL + 1442695040888963407ULL;
			const double unit = static_cast< double >( state >> 11 ) * 0x1.0p-53;
			host[ i ] = 2.0 * unit - 1.0;
		}
		if( v->n > 0 ) {
			SLAB_CUDA( cudaMemcpyAsync( v->d, host.data(), v->n * sizeof( double ), cudaMemcpyHostToDevice,
				v->ctx->stream ) );
			SLAB_CUDA( cudaStreamSynchronize( v->ctx->stream ) );
		}
		if( state_out ) {
			*state_out = state;
		}
	} );
}

int slab_set_all( slab_vec_t v, double value ) {
	return guarded( [ & ] {
		need( v, "set_all" );
		bind( v->ctx );
		op_set_all( v, value );
	} );
}

int slab_dot( slab_vec_t x, slab_vec_t y, double * out ) {
	return guarded( [ & ] {
		need( x, "dot" );
		need( y, "dot" );
		need( out, "dot" );
		same_ctx( x->ctx, y->ctx );
		bind( x->ctx );
		*out = op_dot( x, y );
	} );
}

int slab_waxpby( slab_vec_t w, double alpha, slab_vec_t x, double beta, slab_vec_t y ) {
	return guarded( [ & ] {
		need( w, "waxpby" );
		need( x, "waxpby" );
		need( y, "waxpby" );
		same_ctx( w->ctx, x->ctx );
		same_ctx( w->ctx, y->ctx );
		bind( w->ctx );
		op_waxpby( w, alpha, x, beta, y );
	} );
}

// ---------------------------------------------------------------- matrices

int slab_mat_create_csr( slab_ctx_t ctx, uint64_t nrows, uint64_t ncols, const uint64_t * row_offsets,
	const uint64_t * col_indices, const double * values, slab_mat_t * out ) {
	return guarded( [ & ] {
		need( ctx, "slab_mat_create_csr" );
		need( out, "slab_mat_create_csr" );
		*out = nullptr;
		need( row_offsets, "slab_mat_create_csr" );
		if( row_offsets[ nrows ] > 0 ) {
			need( col_indices, "slab_mat_create_csr" );
			need( values, "slab_mat_create_csr" );
		}
		bind( ctx );
		*out = mat_from_csr( ctx, nrows, ncols, row_offsets, col_indices, values, true );
	} );
}

int slab_mat_create_stencil27( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, slab_mat_t * out ) {
	return guarded( [ & ] {
		need( ctx, "slab_mat_create_stencil27" );
		need( out, "slab_mat_create_stencil27" );
		*out = nullptr;
		bind( ctx );
		*out = mat_stencil27( ctx, nx, ny, nz );
	} );
}

int slab_mat_create_restriction( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, slab_mat_t * out ) {
	return guarded( [ & ] {
		need( ctx, "slab_mat_create_restriction" );
		need( out, "slab_mat_create_restriction" );
		*out = nullptr;
		bind( ctx );
		*out = mat_restriction( ctx, nx, ny, nz );
	} );
}

int slab_mat_destroy( slab_mat_t A ) {
	return guarded( [ & ] {
		if( A ) {
			cudaSetDevice( A->ctx->device );
			cudaStreamSynchronize( A->ctx->stream );
			delete A;
		}
	} );
}

int slab_mat_shape( slab_mat_t A, uint64_t * nrows, uint64_t * ncols, uint64_t * nnz ) {
	return guarded( [ & ] {
		need( A, "slab_mat_shape" );
		if( nrows ) *nrows = A->nrows;
		if( ncols ) *ncols = A->ncols;
		if( nnz ) *nnz = A->nnz;
	} );
}

int slab_mat_download_csr( slab_mat_t A, uint64_t * row_offsets, uint64_t * col_indices, double * values ) {
	return guarded( [ & ] {
		need( A, "slab_mat_download_csr" );
		need( row_offsets, "slab_mat_download_csr" );
		if( A->nnz > 0 ) {
			need( col_indices, "slab_mat_download_csr" );
			need( values, "slab_mat_download_csr" );
		}
		bind( A->ctx );
		mat_download_csr( A, row_offsets, col_indices, values );
	} );
}

int slab_mat_device_bytes( slab_mat_t A, uint64_t * bytes ) {
	return guarded( [ & ] {
		need( A, "slab_mat_device_bytes" );
		need( bytes, "slab_mat_device_bytes" );
		*bytes = A->sell.bytes() + ( A->transposed ? A->transposed->sell.bytes() : 0 );
	} );
}

namespace {
	void fill_format_info( const Sell & S, const BoxTile & T, slab_format_info * out ) {
		out->mask_bytes = T.usable() ? static_cast< uint64_t >( S.nslices ) * kSlice * sizeof( uint32_t ) : 0u;
		out->plane_phases = T.usable() && T.regular ? 1 : 0;
		out->reserved = 0;
		out->packed = S.packed.usable() ? 1 : 0;
		out->width_class = S.packed.ncodes;
		out->dict_size = S.packed.dict_size;
		out->stride = S.packed.stride;
		out->escaped_rows = S.packed.escaped_rows;
		out->plain_bytes = S.bytes();
		out->packed_bytes = S.packed_bytes();
	}
} // namespace

int slab_mat_format_info( slab_mat_t A, slab_format_info * out ) {
	return guarded( [ & ] {
		need( A, "slab_mat_format_info" );
		need( out, "slab_mat_format_info" );
		fill_format_info( A->sell, A->tile, out );
	} );
}

int slab_level_format_info( slab_level_t level, slab_format_info * out ) {
	return guarded( [ & ] {
		need( level, "slab_level_format_info" );
		need( out, "slab_level_format_info" );
		fill_format_info( level->colorA, level->tile, out );
		out->plane_phases = level->planes_ok ? 1 : 0;
	} );
}

// ---------------------------------------------------------------- masks

int slab_mask_create( slab_ctx_t ctx, uint64_t universe, const uint64_t * members, uint64_t count, slab_mask_t * out ) {
	return guarded( [ & ] {
		need( ctx, "slab_mask_create" );
		need( out, "slab_mask_create" );
		*out = nullptr;
		if( count > 0 ) {
			need( members, "slab_mask_create" );
		}
		if( universe >= ( uint64_t( 1 ) << 31 ) ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "IndexMask: universe too large for one device" );
		}
		std::vector< int32_t > m32( count );
		for( uint64_t k = 0; k < count; ++k ) { // index_mask.hpp:41-48
			if( members[ k ] >= universe ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "IndexMask: member out of range" );
			}
			if( k > 0 && members[ k ] <= members[ k - 1 ] ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "IndexMask: members must be strictly increasing" );
			}
			m32[ k ] = static_cast< int32_t >( members[ k ] );
		}
		bind( ctx );
		std::unique_ptr< slab_mask_s > m( new slab_mask_s );
		m->ctx = ctx;
		m->universe = universe;
		m->count = count;
		SLAB_CUDA( cudaMalloc( &m->d_members, std::max< uint64_t >( count, 1 ) * sizeof( int32_t ) ) );
		if( count > 0 ) {
			upload_sync( ctx->stream, m->d_members, m32.data(), count * sizeof( int32_t ) );
		}
		*out = m.release();
	} );
}

int slab_mask_destroy( slab_mask_t m ) {
	return guarded( [ & ] {
		if( m ) {
			cudaSetDevice( m->ctx->device );
			cudaStreamSynchronize( m->ctx->stream );
			delete m;
		}
	} );
}

int slab_mask_info( slab_mask_t m, uint64_t * universe, uint64_t * count ) {
	return guarded( [ & ] {
		need( m, "slab_mask_info" );
		if( universe ) *universe = m->universe;
		if( count ) *count = m->count;
	} );
}

int slab_mxv( slab_vec_t y, slab_mat_t A, slab_vec_t x, unsigned desc ) {
	return guarded( [ & ] {
		need( y, "mxv" );
		need( A, "mxv" );
		need( x, "mxv" );
		same_ctx( A->ctx, y->ctx );
		same_ctx( A->ctx, x->ctx );
		bind( A->ctx );
		op_mxv( y, nullptr, A, x, desc );
	} );
}

int slab_mxv_masked( slab_vec_t y, slab_mask_t mask, slab_mat_t A, slab_vec_t x, unsigned desc ) {
	return guarded( [ & ] {
		need( y, "mxv" );
		need( mask, "mxv" );
		need( A, "mxv" );
		need( x, "mxv" );
		same_ctx( A->ctx, y->ctx );
		same_ctx( A->ctx, x->ctx );
		same_ctx( A->ctx, mask->ctx );
		bind( A->ctx );
		op_mxv( y, mask, A, x, desc );
	} );
}

// ---------------------------------------------------------------- levels

int slab_hierarchy_create( slab_ctx_t ctx, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels, slab_level_t * out ) {
	return guarded( [ & ] {
		need( ctx, "build_hierarchy" );
		need( out, "build_hierarchy" );
		*out = nullptr;
		bind( ctx );
		*out = hierarchy_create( ctx, nx, ny, nz, levels );
	} );
}

int slab_level_create_csr( slab_ctx_t ctx, uint64_t n, const uint64_t * row_offsets, const uint64_t * col_indices,
	const double * values, slab_level_t * out ) {
	return guarded( [ & ] {
		need( ctx, "ProblemLevel" );
		need( out, "ProblemLevel" );
		*out = nullptr;
		need( row_offsets, "ProblemLevel" );
		bind( ctx );
		*out = level_from_csr( ctx, n, row_offsets, col_indices, values );
	} );
}

int slab_level_destroy( slab_level_t level ) {
	return guarded( [ & ] {
		if( level ) {
			cudaSetDevice( level->ctx->device );
			cudaStreamSynchronize( level->ctx->stream );
			spans_discard( level->ctx ); // pending intervals may point into this level's counters
			delete level;
		}
	} );
}

int slab_level_coarser( slab_level_t level, slab_level_t * out ) {
	return guarded( [ & ] {
		need( level, "slab_level_coarser" );
		need( out, "slab_level_coarser" );
		*out = level->coarser.get();
	} );
}

int slab_level_matrix( slab_level_t level, slab_mat_t * A ) {
	return guarded( [ & ] {
		need( level, "slab_level_matrix" );
		need( A, "slab_level_matrix" );
		*A = level->A.get();
	} );
}

int slab_level_restriction( slab_level_t level, slab_mat_t * R ) {
	return guarded( [ & ] {
		need( level, "slab_level_restriction" );
		need( R, "slab_level_restriction" );
		*R = level->R.get();
	} );
}

int slab_level_diag( slab_level_t level, slab_vec_t * a_diag ) {
	return guarded( [ & ] {
		need( level, "slab_level_diag" );
		need( a_diag, "slab_level_diag" );
		*a_diag = level->a_diag.get();
	} );
}

int slab_level_info( slab_level_t level, uint64_t dims[ 3 ], uint64_t * n, uint64_t * nnz, uint64_t * num_colors,
	uint64_t * depth ) {
	return guarded( [ & ] {
		need( level, "slab_level_info" );
		if( dims ) {
			std::memcpy( dims, level->dims, sizeof( level->dims ) );
		}
		if( n ) *n = level->n;
		if( nnz ) *nnz = level->nnz;
		if( num_colors ) *num_colors = level->num_colors;
		if( depth ) {
			uint64_t d = 0;
			for( slab_level_s * at = level; at; at = at->coarser.get() ) {
				++d;
			}
			*depth = d;
		}
	} );
}

int slab_level_color_info( slab_level_t level, uint64_t k, uint64_t * size, uint64_t * color_nnz ) {
	return guarded( [ & ] {
		need( level, "slab_level_color_info" );
		if( k >= level->num_colors ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "colour index out of range" );
		}
		if( size ) *size = level->color_size[ k ];
		if( color_nnz ) *color_nnz = level->color_nnz[ k ];
	} );
}

int slab_level_color_members( slab_level_t level, uint64_t k, uint64_t * members ) {
	return guarded( [ & ] {
		need( level, "slab_level_color_members" );
		if( k >= level->num_colors ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "colour index out of range" );
		}
		const uint64_t size = level->color_size[ k ];
		if( size == 0 ) {
			return;
		}
		need( members, "slab_level_color_members" );
		bind( level->ctx );
		std::vector< int32_t > rows( size );
		SLAB_CUDA( cudaStreamSynchronize( level->ctx->stream ) );
		SLAB_CUDA( cudaMemcpy( rows.data(), level->d_rows + level->color_pos[ k ], size * sizeof( int32_t ),
			cudaMemcpyDeviceToHost ) );
		for( uint64_t q = 0; q < size; ++q ) {
			members[ q ] = static_cast< uint64_t >( rows[ q ] );
		}
	} );
}

int slab_level_stats_get( slab_level_t level, slab_level_stats * out ) {
	return guarded( [ & ] {
		need( level, "slab_level_stats_get" );
		need( out, "slab_level_stats_get" );
		bind( level->ctx );
		spans_resolve( level->ctx ); // pending device-time intervals land in the counters now
		*out = level->stats;
	} );
}

int slab_level_stats_reset( slab_level_t level ) {
	return guarded( [ & ] {
		need( level, "slab_level_stats_reset" );
		bind( level->ctx );
		spans_resolve( level->ctx );
		for( slab_level_s * at = level; at; at = at->coarser.get() ) {
			at->stats = slab_level_stats{};
		}
	} );
}

// ---------------------------------------------------------------- smoother / multigrid

#define SLAB_LEVEL_ZR( name )                  \
	need( level, name );                       \
	need( z, name );                           \
	need( r, name );                           \
	same_ctx( level->ctx, z->ctx );            \
	same_ctx( level->ctx, r->ctx );            \
	bind( level->ctx )

int slab_rbgs_color_step( slab_level_t level, uint64_t k, slab_vec_t z, slab_vec_t r ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "rbgs_color_step" );
		rbgs_color_step( level, k, z, r );
	} );
}

int slab_rbgs_color_step_twice( slab_level_t level, uint64_t k, slab_vec_t z, slab_vec_t r ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "rbgs_color_step_twice" );
		rbgs_color_step_twice( level, k, z, r );
	} );
}

int slab_rbgs_forward( slab_level_t level, slab_vec_t z, slab_vec_t r ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "rbgs_forward" );
		rbgs_forward( level, z, r );
	} );
}

int slab_rbgs_backward( slab_level_t level, slab_vec_t z, slab_vec_t r ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "rbgs_backward" );
		rbgs_backward( level, z, r );
	} );
}

int slab_rbgs_symmetric( slab_level_t level, slab_vec_t z, slab_vec_t r, uint64_t sweeps ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "rbgs_symmetric" );
		rbgs_symmetric( level, z, r, sweeps );
	} );
}

int slab_restrict_vector( slab_level_t level, slab_vec_t v_fine, slab_vec_t out ) {
	return guarded( [ & ] {
		need( level, "restrict_vector" );
		need( v_fine, "restrict_vector" );
		need( out, "restrict_vector" );
		same_ctx( level->ctx, v_fine->ctx );
		same_ctx( level->ctx, out->ctx );
		bind( level->ctx );
		restrict_vector( level, v_fine, out );
	} );
}

int slab_refine_and_add( slab_level_t level, slab_vec_t z, slab_vec_t z_c ) {
	return guarded( [ & ] {
		need( level, "refine_and_add" );
		need( z, "refine_and_add" );
		need( z_c, "refine_and_add" );
		same_ctx( level->ctx, z->ctx );
		same_ctx( level->ctx, z_c->ctx );
		bind( level->ctx );
		refine_and_add( level, z, z_c );
	} );
}

int slab_mg_vcycle( slab_level_t level, slab_vec_t z, slab_vec_t r, uint64_t sweeps ) {
	return guarded( [ & ] {
		SLAB_LEVEL_ZR( "mg_vcycle" );
		mg_vcycle( level, z, r, sweeps );
	} );
}

// ---------------------------------------------------------------- cg

void slab_cg_config_default( slab_cg_config * cfg ) {
	if( cfg ) {
		cfg->max_iters = 500;
		cfg->rtol = 1e-6;
		cfg->use_preconditioner = 1;
		cfg->has_fixed_iterations = 0;
		cfg->fixed_iterations = 0;
		cfg->sweeps = 1;
	}
}

int slab_cg_solve( slab_level_t hierarchy, slab_vec_t b, slab_vec_t x0, const slab_cg_config * cfg, slab_vec_t x,
	double * history, slab_cg_result * result ) {
	return guarded( [ & ] {
		need( hierarchy, "cg_solve" );
		need( b, "cg_solve" );
		need( x0, "cg_solve" );
		need( x, "cg_solve" );
		need( cfg, "cg_solve" );
		need( history, "cg_solve" );
		same_ctx( hierarchy->ctx, b->ctx );
		same_ctx( hierarchy->ctx, x0->ctx );
		same_ctx( hierarchy->ctx, x->ctx );
		bind( hierarchy->ctx );
		cg_solve( hierarchy, b, x0, cfg, x, history, result );
	} );
}

int slab_cg_solve_host( slab_level_t hierarchy, const double * b, const double * x0, uint64_t n,
	const slab_cg_config * cfg, double * x, double * history, slab_cg_result * result ) {
	return guarded( [ & ] {
		need( hierarchy, "cg_solve" );
		need( cfg, "cg_solve" );
		need( history, "cg_solve" );
		if( n != hierarchy->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "cg_solve: vector lengths differ from the system size" );
		}
		if( n > 0 ) {
			need( b, "cg_solve" );
			need( x0, "cg_solve" );
			need( x, "cg_solve" );
		}
		bind( hierarchy->ctx );
		cg_solve_host( hierarchy, b, x0, cfg, x, history, result );
	} );
}

int slab_residual_norm( slab_mat_t A, slab_vec_t x, slab_vec_t b, double * out ) {
	return guarded( [ & ] {
		need( A, "residual_norm" );
		need( x, "residual_norm" );
		need( b, "residual_norm" );
		need( out, "residual_norm" );
		same_ctx( A->ctx, x->ctx );
		same_ctx( A->ctx, b->ctx );
		bind( A->ctx );
		*out = residual_norm( A, x, b );
	} );
}

// ---------------------------------------------------------------- domain decomposition

int slab_ctx_set_process_grid( slab_ctx_t ctx, int px, int py, int pz, int rank ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_set_process_grid" );
		dist_set_grid( ctx, px, py, pz, rank );
	} );
}

int slab_nccl_unique_id( unsigned char * out128 ) {
	return guarded( [ & ] {
		need( out128, "slab_nccl_unique_id" );
		NcclUniqueId id;
		nccl_unique_id( &id );
		std::memcpy( out128, id.internal, sizeof( id.internal ) );
	} );
}

int slab_ctx_init_nccl( slab_ctx_t ctx, const unsigned char * id128 ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_init_nccl" );
		need( id128, "slab_ctx_init_nccl" );
		bind( ctx );
		NcclUniqueId id;
		std::memcpy( id.internal, id128, sizeof( id.internal ) );
		dist_init_nccl( ctx, &id );
	} );
}

int slab_ctx_dist_info( slab_ctx_t ctx, int grid[ 3 ], int * rank, int * nranks, int * has_comm, uint64_t * exchanges ) {
	return guarded( [ & ] {
		need( ctx, "slab_ctx_dist_info" );
		const DistState * d = ctx->dist;
		if( grid ) {
			for( int a = 0; a < 3; ++a ) {
				grid[ a ] = d ? d->p[ a ] : 1;
			}
		}
		if( rank ) *rank = d ? d->rank : 0;
		if( nranks ) *nranks = d ? d->nranks : 1;
		if( has_comm ) *has_comm = d && d->comm ? 1 : 0;
		if( exchanges ) *exchanges = d ? d->exchanges : 0;
	} );
}

int slab_level_decomp( slab_level_t level, uint64_t global_dims[ 3 ], uint64_t offset[ 3 ], uint64_t * n_ghost ) {
	return guarded( [ & ] {
		need( level, "slab_level_decomp" );
		for( int a = 0; a < 3; ++a ) {
			if( global_dims ) global_dims[ a ] = static_cast< uint64_t >( level->decomp.g[ a ] );
			if( offset ) offset[ a ] = static_cast< uint64_t >( level->decomp.o[ a ] );
		}
		if( n_ghost ) *n_ghost = static_cast< uint64_t >( level->decomp.n_ghost );
	} );
}

namespace {
	void halo_range( slab_level_s * level, int dir, int color, int & send_first, int & send_n, int & recv_first, int & recv_n ) {
		if( level->plan == nullptr ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "level is not distributed" );
		}
		if( dir < 0 || dir >= 27 || color < -1 || color >= 8 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "halo: direction must be in [0,27), colour in [-1,8)" );
		}
		const HaloPlan * plan = level->plan;
		const int c0 = color < 0 ? 0 : color, c1 = color < 0 ? 8 : color + 1;
		send_first = plan->send_off[ dir ][ c0 ];
		recv_first = plan->D.ghost_base[ dir ][ c0 ];
		send_n = recv_n = 0;
		for( int c = c0; c < c1; ++c ) {
			send_n += plan->send_count[ dir ][ c ];
			recv_n += plan->D.ghost_count[ dir ][ c ];
		}
	}
} // namespace

int slab_level_halo_info( slab_level_t level, int dir, int color, uint64_t * send_count, uint64_t * recv_count, int * peer ) {
	return guarded( [ & ] {
		need( level, "slab_level_halo_info" );
		int sf, sn, rf, rn;
		halo_range( level, dir, color, sf, sn, rf, rn );
		if( send_count ) *send_count = static_cast< uint64_t >( sn );
		if( recv_count ) *recv_count = static_cast< uint64_t >( rn );
		if( peer ) *peer = level->plan->peer[ dir ];
	} );
}

int slab_level_halo_pack( slab_level_t level, slab_vec_t v, int dir, int color, double * host_out ) {
	return guarded( [ & ] {
		need( level, "slab_level_halo_pack" );
		need( v, "slab_level_halo_pack" );
		int sf, sn, rf, rn;
		halo_range( level, dir, color, sf, sn, rf, rn );
		if( v->n != level->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "halo: vector length differs from the level size" );
		}
		if( sn == 0 ) {
			return;
		}
		need( host_out, "slab_level_halo_pack" );
		slab_ctx_s * ctx = level->ctx;
		bind( ctx );
		halo_pack( ctx, level->plan, v, color );
		SLAB_CUDA( cudaMemcpyAsync( host_out, level->plan->d_sendbuf + sf, static_cast< size_t >( sn ) * sizeof( double ),
			cudaMemcpyDeviceToHost, ctx->stream ) );
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
	} );
}

int slab_level_halo_unpack( slab_level_t level, slab_vec_t v, int dir, int color, const double * host_in ) {
	return guarded( [ & ] {
		need( level, "slab_level_halo_unpack" );
		need( v, "slab_level_halo_unpack" );
		int sf, sn, rf, rn;
		halo_range( level, dir, color, sf, sn, rf, rn );
		if( v->n != level->n
			|| v->n_alloc < static_cast< uint64_t >( level->decomp.n_local ) + static_cast< uint64_t >( level->decomp.n_ghost ) ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "halo: vector does not belong to this level (or predates the hierarchy)" );
		}
		if( rn == 0 ) {
			return;
		}
		need( host_in, "slab_level_halo_unpack" );
		bind( level->ctx );
		upload_sync( level->ctx->stream, v->d + level->decomp.n_local + rf, host_in, static_cast< size_t >( rn ) * sizeof( double ) );
	} );
}

// host-only: the halo plan of one rank, computed without touching a GPU
int slab_plan_query( const uint64_t local_dims[ 3 ], const uint64_t grid[ 3 ], uint64_t rank, int dir, int color,
	uint64_t * n_local, uint64_t * n_ghost, uint64_t * send_count, uint64_t * recv_count, int64_t * peer,
	uint64_t * ghost_base, uint64_t * send_indices ) {
	return guarded( [ & ] {
		need( local_dims, "slab_plan_query" );
		need( grid, "slab_plan_query" );
		const int p[ 3 ] = { static_cast< int >( grid[ 0 ] ), static_cast< int >( grid[ 1 ] ), static_cast< int >( grid[ 2 ] ) };
		const int l[ 3 ] = { static_cast< int >( local_dims[ 0 ] ), static_cast< int >( local_dims[ 1 ] ),
			static_cast< int >( local_dims[ 2 ] ) };
		if( p[ 0 ] < 1 || p[ 1 ] < 1 || p[ 2 ] < 1 || rank >= static_cast< uint64_t >( p[ 0 ] ) * p[ 1 ] * p[ 2 ] || dir < 0 || dir >= 27
			|| color < 0 || color >= 8 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "slab_plan_query: bad grid, rank, direction or colour" );
		}
		int r[ 3 ];
		rank_coords( p, static_cast< int >( rank ), r );
		const Decomp D = make_decomp( l, p, r );
		const int d[ 3 ] = { dir % 3 - 1, ( dir / 3 ) % 3 - 1, dir / 9 - 1 };
		const int nr[ 3 ] = { r[ 0 ] + d[ 0 ], r[ 1 ] + d[ 1 ], r[ 2 ] + d[ 2 ] };
		const bool exists = dir != 13 && nr[ 0 ] >= 0 && nr[ 0 ] < p[ 0 ] && nr[ 1 ] >= 0 && nr[ 1 ] < p[ 1 ] && nr[ 2 ] >= 0
			&& nr[ 2 ] < p[ 2 ];
		std::vector< int32_t > list;
		if( exists ) {
			send_list( D, dir, color, list );
		}
		if( n_local ) *n_local = static_cast< uint64_t >( D.n_local );
		if( n_ghost ) *n_ghost = static_cast< uint64_t >( D.n_ghost );
		if( send_count ) *send_count = list.size();
		if( recv_count ) *recv_count = static_cast< uint64_t >( D.ghost_count[ dir ][ color ] );
		if( peer ) *peer = exists ? nr[ 0 ] + p[ 0 ] * ( nr[ 1 ] + p[ 1 ] * nr[ 2 ] ) : -1;
		if( ghost_base ) *ghost_base = static_cast< uint64_t >( D.ghost_base[ dir ][ color ] );
		if( send_indices ) {
			for( size_t k = 0; k < list.size(); ++k ) {
				send_indices[ k ] = static_cast< uint64_t >( list[ k ] );
			}
		}
	} );
}

int slab_plan_local_index( const uint64_t local_dims[ 3 ], const uint64_t grid[ 3 ], uint64_t rank, uint64_t X, uint64_t Y,
	uint64_t Z, int64_t * out ) {
	return guarded( [ & ] {
		need( local_dims, "slab_plan_local_index" );
		need( grid, "slab_plan_local_index" );
		need( out, "slab_plan_local_index" );
		const int p[ 3 ] = { static_cast< int >( grid[ 0 ] ), static_cast< int >( grid[ 1 ] ), static_cast< int >( grid[ 2 ] ) };
		const int l[ 3 ] = { static_cast< int >( local_dims[ 0 ] ), static_cast< int >( local_dims[ 1 ] ),
			static_cast< int >( local_dims[ 2 ] ) };
		int r[ 3 ];
		rank_coords( p, static_cast< int >( rank ), r );
		const Decomp D = make_decomp( l, p, r );
		const int c[ 3 ] = { static_cast< int >( X ), static_cast< int >( Y ), static_cast< int >( Z ) };
		for( int a = 0; a < 3; ++a ) { // only points within one layer of the owned box are addressable
			if( c[ a ] < 0 || c[ a ] >= D.g[ a ] || c[ a ] < D.o[ a ] - 1 || c[ a ] > D.o[ a ] + D.l[ a ] ) {
				*out = -1;
				return;
			}
		}
		*out = local_index( D, c[ 0 ], c[ 1 ], c[ 2 ] );
	} );
}

} // extern "C"
