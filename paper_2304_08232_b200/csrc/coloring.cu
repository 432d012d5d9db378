// coloring.cu — greedy_color (coloring.hpp:114-158) on the device, for general square matrices.
//
// The reference colours the rows in increasing index order: a row takes the smallest colour that none of its already
// coloured neighbours has, neighbours being the columns of the row in A united with its column in A^T (so
// non-symmetric patterns are handled too). "Already coloured" means "lower index", so the result is a pure function
// of the pattern: colour(i) = mex{ colour(j) : j < i, j ~ i }. That recurrence is evaluated here as a wavefront —
// a row colours itself as soon as all its lower neighbours have their colours — which reproduces the sequential
// result exactly, whatever the timing:
//   * thread blocks take tickets (an atomic counter), so block t owns rows [256 t, 256 t + 256) and every block with a
//     lower ticket is resident or finished: waiting on lower rows can never deadlock;
//   * inside a block the rows advance in rounds separated by block barriers, the block's colours in shared memory;
//     rows of lower blocks are read from global memory (written with a device-scope fence) and simply make the row
//     wait another round while they are unset.
// The transpose pattern is built on the device as well (count, cub scan, fill — the order inside a list does not
// matter to a set). The colour of every row comes back to the host once; grouping the rows by colour (ascending
// inside a colour, coloring.hpp:148-151) happens where the colour-major SELL copy is assembled from the host CSR.
#include <cstdint>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"
#include "kernels.cuh"

namespace slabgpu {

	namespace {

		constexpr int kRowsPerBlock = 256;
		constexpr int32_t kUnset = -1;

		__global__ void k_transpose_count( const int64_t * __restrict__ ro, const int32_t * __restrict__ co, int64_t n, int32_t * __restrict__ count ) {
			const int64_t i = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
			if( i >= n ) {
				return;
			}
			for( int64_t k = ro[ i ]; k < ro[ i + 1 ]; ++k ) {
				if( co[ k ] != i ) {
					atomicAdd( count + co[ k ], 1 );
				}
			}
		}

		__global__ void k_transpose_fill( const int64_t * __restrict__ ro, const int32_t * __restrict__ co, int64_t n, const int64_t * __restrict__ t_off,
			int32_t * __restrict__ cursor, int32_t * __restrict__ t_idx ) {
			const int64_t i = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
			if( i >= n ) {
				return;
			}
			for( int64_t k = ro[ i ]; k < ro[ i + 1 ]; ++k ) {
				const int32_t j = co[ k ];
				if( j != i ) {
					t_idx[ t_off[ j ] + atomicAdd( cursor + j, 1 ) ] = static_cast< int32_t >( i );
				}
			}
		}

		__device__ __forceinline__ int32_t load_color( const int32_t * color, int64_t j ) {
			int32_t c;
			asm volatile( "ld.acquire.gpu.global.s32 %0, [%1];" : "=r"( c ) : "l"( color + j ) : "memory" );
			return c;
		}

		// colour(i) = smallest colour no lower-index neighbour has (coloring.hpp:131-143)
		__global__ void __launch_bounds__( kRowsPerBlock ) k_greedy_wavefront( const int64_t * __restrict__ ro, const int32_t * __restrict__ co,
			const int64_t * __restrict__ t_off, const int32_t * __restrict__ t_idx, int64_t n, int32_t * color, unsigned int * ticket_counter ) {
			__shared__ int32_t s_color[ kRowsPerBlock ];
			__shared__ unsigned int s_ticket;
			if( threadIdx.x == 0 ) {
				s_ticket = atomicAdd( ticket_counter, 1u );
			}
			s_color[ threadIdx.x ] = kUnset;
			__syncthreads();
			const int64_t base = static_cast< int64_t >( s_ticket ) * kRowsPerBlock;
			const int64_t i = base + threadIdx.x;
			bool done = i >= n;
			int32_t mine = kUnset;
			const int64_t a0 = done ? 0 : ro[ i ], a1 = done ? 0 : ro[ i + 1 ];
			const int64_t b0 = done ? 0 : t_off[ i ], b1 = done ? 0 : t_off[ i + 1 ];
			while( true ) {
				bool ready = !done;
				uint64_t taken[ 4 ] = { 0, 0, 0, 0 }; // colours below 256 that a lower neighbour has
				bool beyond = false;                  // ... and whether one has a colour from 256 on
				const auto visit = [ & ]( int64_t j ) {
					if( j >= i ) {
						return;
					}
					const int32_t c = j >= base ? s_color[ j - base ] : load_color( color, j );
					if( c == kUnset ) {
						ready = false;
					} else if( c < 256 ) {
						taken[ c >> 6 ] |= uint64_t( 1 ) << ( c & 63 );
					} else {
						beyond = true;
					}
				};
				if( !done ) {
					for( int64_t k = a0; k < a1 && ready; ++k ) {
						visit( co[ k ] );
					}
					for( int64_t k = b0; k < b1 && ready; ++k ) {
						visit( t_idx[ k ] );
					}
				}
				int32_t pick = kUnset;
				if( ready ) {
					for( int w = 0; w < 4 && pick == kUnset; ++w ) {
						if( ~taken[ w ] != 0 ) {
							pick = 64 * w + __ffsll( static_cast< long long >( ~taken[ w ] ) ) - 1;
						}
					}
					if( pick == kUnset ) { // 256 colours taken: search upwards by membership (rows of degree >= 256 only)
						pick = 256;
						bool hit = beyond;
						while( hit ) {
							hit = false;
							const auto has = [ & ]( int64_t j ) {
								if( j < i && ( j >= base ? s_color[ j - base ] : load_color( color, j ) ) == pick ) {
									hit = true;
								}
							};
							for( int64_t k = a0; k < a1 && !hit; ++k ) {
								has( co[ k ] );
							}
							for( int64_t k = b0; k < b1 && !hit; ++k ) {
								has( t_idx[ k ] );
							}
							if( hit ) {
								++pick;
							}
						}
					}
				}
				__syncthreads(); // every read of this round's shared colours is done
				if( ready ) {
					mine = pick;
					s_color[ threadIdx.x ] = pick;
					done = true;
				}
				if( __syncthreads_and( done ? 1 : 0 ) ) {
					break;
				}
			}
			if( i < n ) {
				color[ i ] = mine;
			}
			__threadfence(); // blocks with higher tickets read these colours
		}

	} // namespace

	// color[i] for every row, and the number of colours; ro / co are the host CSR of a square matrix (validated by
	// the caller), n < 2^31
	void greedy_color_device( slab_ctx_s * ctx, uint64_t n, const uint64_t * ro, const uint64_t * co, std::vector< int32_t > & color,
		uint64_t & num_colors ) {
		using namespace kern::dev;
		color.assign( n, 0 );
		num_colors = 0;
		if( n == 0 ) {
			return;
		}
		const uint64_t nnz = ro[ n ];
		cudaStream_t st = ctx->stream;
		std::vector< int64_t > h_ro( ro, ro + n + 1 );
		std::vector< int32_t > h_co( nnz );
		for( uint64_t k = 0; k < nnz; ++k ) {
			h_co[ k ] = static_cast< int32_t >( co[ k ] );
		}
		int64_t * d_ro = nullptr, * d_toff = nullptr;
		int32_t * d_co = nullptr, * d_cnt = nullptr, * d_tidx = nullptr, * d_color = nullptr;
		unsigned int * d_ticket = nullptr;
		void * d_tmp = nullptr;
		const auto release = [ & ]() {
			cudaFree( d_ro );
			cudaFree( d_toff );
			cudaFree( d_co );
			cudaFree( d_cnt );
			cudaFree( d_tidx );
			cudaFree( d_color );
			cudaFree( d_ticket );
			cudaFree( d_tmp );
		};
		try {
			SLAB_CUDA( cudaMalloc( &d_ro, ( n + 1 ) * sizeof( int64_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_toff, ( n + 1 ) * sizeof( int64_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_co, std::max< uint64_t >( nnz, 1 ) * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_cnt, ( n + 1 ) * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_tidx, std::max< uint64_t >( nnz, 1 ) * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_color, n * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_ticket, sizeof( unsigned int ) ) );
			upload_sync( st, d_ro, h_ro.data(), ( n + 1 ) * sizeof( int64_t ) );
			if( nnz > 0 ) {
				upload_sync( st, d_co, h_co.data(), nnz * sizeof( int32_t ) );
			}
			SLAB_CUDA( cudaMemsetAsync( d_cnt, 0, ( n + 1 ) * sizeof( int32_t ), st ) );
			SLAB_CUDA( cudaMemsetAsync( d_ticket, 0, sizeof( unsigned int ), st ) );
			SLAB_CUDA( cudaMemsetAsync( d_color, 0xff, n * sizeof( int32_t ), st ) ); // kUnset
			const unsigned int grid = blocks_for( n );
			k_transpose_count<<< grid, kBlock, 0, st >>>( d_ro, d_co, static_cast< int64_t >( n ), d_cnt );
			SLAB_CUDA( cudaGetLastError() );
			count_launch();
			size_t tmp_bytes = 0;
			SLAB_CUDA( cub::DeviceScan::ExclusiveSum( nullptr, tmp_bytes, d_cnt, d_toff, static_cast< int >( n + 1 ), st ) );
			SLAB_CUDA( cudaMalloc( &d_tmp, std::max< size_t >( tmp_bytes, 16 ) ) );
			SLAB_CUDA( cub::DeviceScan::ExclusiveSum( d_tmp, tmp_bytes, d_cnt, d_toff, static_cast< int >( n + 1 ), st ) );
			count_launch();
			SLAB_CUDA( cudaMemsetAsync( d_cnt, 0, ( n + 1 ) * sizeof( int32_t ), st ) ); // now the fill cursors
			k_transpose_fill<<< grid, kBlock, 0, st >>>( d_ro, d_co, static_cast< int64_t >( n ), d_toff, d_cnt, d_tidx );
			SLAB_CUDA( cudaGetLastError() );
			count_launch();
			const unsigned int cgrid = static_cast< unsigned int >( ( n + kRowsPerBlock - 1 ) / kRowsPerBlock );
			k_greedy_wavefront<<< cgrid, kRowsPerBlock, 0, st >>>( d_ro, d_co, d_toff, d_tidx, static_cast< int64_t >( n ), d_color, d_ticket );
			SLAB_CUDA( cudaGetLastError() );
			count_launch();
			SLAB_CUDA( cudaMemcpyAsync( color.data(), d_color, n * sizeof( int32_t ), cudaMemcpyDeviceToHost, st ) );
			SLAB_CUDA( cudaStreamSynchronize( st ) );
		} catch( ... ) {
			release();
			throw;
		}
		release();
		for( uint64_t i = 0; i < n; ++i ) {
			if( color[ i ] < 0 ) {
				fail( SLAB_ERR_INTERNAL, "greedy_color: a row was left without a colour" );
			}
			num_colors = std::max< uint64_t >( num_colors, static_cast< uint64_t >( color[ i ] ) + 1 );
		}
	}

} // namespace slabgpu
