// kernels.cu — hand-written sm_100a kernels of the CG+MG hot path.
//
// Arithmetic contract: the reference is compiled without FMA
// (proj/CMakeLists.txt:8-14), so every product is rounded before it is added. All fp64
// arithmetic below goes through __dmul_rn/__dadd_rn/__ddiv_rn, which the compiler never
// contracts, and the file is additionally built with -fmad=false.
//
// All kernels are HBM-bound streaming kernels: the matrix is read once, coalesced, with a
// streaming (evict-first) hint so that it does not push the vectors out of the 126 MB L2; the
// vector gathers are served by L1/L2.
#include "kernels.cuh"

#include <cuda_runtime.h>

#include "common.hpp"

namespace slabgpu {

	uint64_t g_launch_count = 0;

	namespace kern {

		namespace {

			constexpr int kBlock = 256;

			inline unsigned int blocks_for( uint64_t count, int block = kBlock ) {
				return static_cast< unsigned int >( ( count + block - 1 ) / block );
			}

			// ordered row sum over one SELL row: acc = acc + val*x[col], stored entries only,
			// ascending column order (operations.hpp:116-125). `diag_row` >= 0 also extracts
			// the stored diagonal (problem.hpp:143-166) on the way.
			template< bool WANT_DIAG >
			__device__ __forceinline__ double sell_row_sum( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, int64_t pos, const double * x,
				int32_t diag_row, double & diag ) {
				const int64_t s = pos >> 5;
				const int lane = static_cast< int >( pos & 31 );
				const int64_t begin = slice_off[ s ] + lane;
				const int64_t end = slice_off[ s + 1 ];
				double acc = 0.0;
				#pragma unroll 9
				for( int64_t e = begin; e < end; e += kSlice ) {
					const int32_t c = __ldcs( cols + e );
					const double v = __ldcs( vals + e );
					const double xv = x[ c < 0 ? 0 : c ];
					const double sum = __dadd_rn( acc, __dmul_rn( v, xv ) );
					acc = c < 0 ? acc : sum;
					if( WANT_DIAG ) {
						diag = c == diag_row ? v : diag;
					}
				}
				return acc;
			}

			// ------------------------------------------------------------ vector ops

			__global__ void k_fill( double * __restrict__ v, uint64_t n, double value ) {
				const uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( i < n ) {
					v[ i ] = value;
				}
			}

			// operations.hpp:103 — w may alias x or y: each thread reads its inputs before writing
			__global__ void k_waxpby( double * w, double alpha, const double * x, double beta, const double * y,
				uint64_t n ) {
				const uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( i < n ) {
					const double ax = __dmul_rn( alpha, x[ i ] );
					const double by = __dmul_rn( beta, y[ i ] );
					w[ i ] = __dadd_rn( ax, by );
				}
			}

			// operations.hpp:61-91: one warp per 4096-element chunk. The 32 lanes form the rounded
			// products in parallel (coalesced), lane 0 then adds them left to right; the block that
			// finishes last adds the per-chunk partials in chunk order.
			__global__ void __launch_bounds__( 32 ) k_dot_exact( const double * __restrict__ x,
				const double * __restrict__ y, uint64_t n, double * partials, unsigned int * counter, double * out ) {
				__shared__ double prod[ kDotChunk ];
				const uint64_t begin = static_cast< uint64_t >( blockIdx.x ) * kDotChunk;
				const uint64_t remaining = n - begin;
				const int len = static_cast< int >( remaining < kDotChunk ? remaining : kDotChunk );
				const int lane = threadIdx.x;
				for( int i = lane; i < len; i += 32 ) {
					prod[ i ] = __dmul_rn( x[ begin + i ], y[ begin + i ] );
				}
				__syncwarp();
				if( lane == 0 ) {
					double acc = 0.0;
					#pragma unroll 16
					for( int i = 0; i < len; ++i ) {
						acc = __dadd_rn( acc, prod[ i ] );
					}
					partials[ blockIdx.x ] = acc;
					__threadfence();
					const unsigned int ticket = atomicAdd( counter, 1u );
					if( ticket == gridDim.x - 1 ) {
						__threadfence();
						double total = 0.0;
						for( unsigned int c = 0; c < gridDim.x; ++c ) {
							total = __dadd_rn( total, __ldcg( partials + c ) );
						}
						*out = total;
						*counter = 0u;
					}
				}
			}

			__global__ void k_dot_empty( double * out ) {
				*out = 0.0;
			}

			// fixed-shape tree reduction: grid-stride partial per thread, shuffle tree per warp,
			// shared-memory tree per block, last block folds the block partials the same way.
			__device__ __forceinline__ double block_tree_sum( double v, double * smem ) {
				#pragma unroll
				for( int off = 16; off > 0; off >>= 1 ) {
					v = __dadd_rn( v, __shfl_down_sync( 0xffffffffu, v, off ) );
				}
				const int warp = threadIdx.x >> 5;
				const int lane = threadIdx.x & 31;
				if( lane == 0 ) {
					smem[ warp ] = v;
				}
				__syncthreads();
				const int nwarps = blockDim.x >> 5;
				v = threadIdx.x < nwarps ? smem[ threadIdx.x ] : 0.0;
				if( warp == 0 ) {
					#pragma unroll
					for( int off = 16; off > 0; off >>= 1 ) {
						v = __dadd_rn( v, __shfl_down_sync( 0xffffffffu, v, off ) );
					}
				}
				__syncthreads();
				return v; // valid in thread 0
			}

			__global__ void __launch_bounds__( kBlock ) k_dot_tree( const double * __restrict__ x,
				const double * __restrict__ y, uint64_t n, double * partials, unsigned int * counter, double * out ) {
				__shared__ double smem[ 32 ];
				__shared__ bool is_last;
				double acc = 0.0;
				const uint64_t stride = static_cast< uint64_t >( gridDim.x ) * blockDim.x;
				for( uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x; i < n; i += stride ) {
					acc = __dadd_rn( acc, __dmul_rn( x[ i ], y[ i ] ) );
				}
				acc = block_tree_sum( acc, smem );
				if( threadIdx.x == 0 ) {
					partials[ blockIdx.x ] = acc;
					__threadfence();
					const unsigned int ticket = atomicAdd( counter, 1u );
					is_last = ticket == gridDim.x - 1;
				}
				__syncthreads();
				if( is_last ) {
					__threadfence();
					double v = 0.0;
					for( unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x ) {
						v = __dadd_rn( v, __ldcg( partials + b ) );
					}
					v = block_tree_sum( v, smem );
					if( threadIdx.x == 0 ) {
						*out = v;
						*counter = 0u;
					}
				}
			}

			// ------------------------------------------------------------ SELL products

			__global__ void __launch_bounds__( kBlock ) k_spmv( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const double * __restrict__ x,
				double * __restrict__ y, int64_t nrows ) {
				const int64_t row = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( row >= nrows ) {
					return;
				}
				double unused = 0.0;
				y[ row ] = sell_row_sum< false >( slice_off, vals, cols, row, x, -1, unused );
			}

			__global__ void __launch_bounds__( kBlock ) k_spmv_masked( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const double * __restrict__ x,
				double * __restrict__ y, const int32_t * __restrict__ members, int64_t count ) {
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( k >= count ) {
					return;
				}
				const int64_t row = members[ k ];
				double unused = 0.0;
				y[ row ] = sell_row_sum< false >( slice_off, vals, cols, row, x, -1, unused );
			}

			// smoother.hpp:60-72 fused: s = row sum over z, then z[i] = ((r[i] - s) + z[i]*d) / d.
			// Rows of one colour never neighbour each other, so reading z while other threads of
			// the same launch write their own z[i] is race-free (coloring.hpp:165-204).
			__global__ void __launch_bounds__( kBlock ) k_gs_color( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t pos_begin, int64_t pos_count, double * z, const double * __restrict__ r ) {
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( k >= pos_count ) {
					return;
				}
				const int64_t pos = pos_begin + k;
				const int32_t i = rows[ pos ];
				if( i < 0 ) {
					return;
				}
				double d = 0.0;
				const double s = sell_row_sum< true >( slice_off, vals, cols, pos, z, i, d );
				const double zi = z[ i ];
				const double ri = r[ i ];
				z[ i ] = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -s ), __dmul_rn( zi, d ) ), d );
			}

			// multigrid.hpp:100-104 fused on the injected rows (= the colour-0 block, whose p-th
			// member is the fine point of coarse index p): f = 1*r + (-1)*(A z), r_c = 0 + 1*f.
			__global__ void __launch_bounds__( kBlock ) k_residual_restrict( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t n_coarse, const double * __restrict__ z, const double * __restrict__ r,
				double * __restrict__ r_c ) {
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( p >= n_coarse ) {
					return;
				}
				const int32_t i = rows[ p ];
				double unused = 0.0;
				const double az = sell_row_sum< false >( slice_off, vals, cols, p, z, -1, unused );
				const double f = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -1.0, az ) );
				r_c[ p ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
			}

			// multigrid.hpp:71-81 at the injected rows: f[i] = 0 + 1*z_c[p]; z[i] = 1*z[i] + 1*f[i].
			// (Elsewhere the reference computes z + 0.0, which only turns -0.0 into +0.0.)
			__global__ void k_prolong_add( const int32_t * __restrict__ rows, int64_t n_coarse, double * z,
				const double * __restrict__ z_c ) {
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( p >= n_coarse ) {
					return;
				}
				const int32_t i = rows[ p ];
				const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, z_c[ p ] ) );
				z[ i ] = __dadd_rn( __dmul_rn( 1.0, z[ i ] ), __dmul_rn( 1.0, f ) );
			}

			// ------------------------------------------------------------ CG updates

			__global__ void k_cg_update_p( double * p, const double * __restrict__ z, const double * __restrict__ scalars,
				const unsigned int * __restrict__ iter_counter, uint64_t n ) {
				const uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( i >= n ) {
					return;
				}
				const double zi = z[ i ];
				if( *iter_counter == 0u ) { // cg.hpp:118  waxpby( p, 1.0, z, 0.0, z )
					p[ i ] = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 0.0, zi ) );
				} else {      // cg.hpp:120  waxpby( p, 1.0, z, rho / rho_prev, p )
					const double beta = __ddiv_rn( scalars[ S_RHO ], scalars[ S_RHO_PREV ] );
					p[ i ] = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( beta, p[ i ] ) );
				}
			}

			__global__ void k_cg_update_xr( double * x, double * r, const double * __restrict__ p,
				const double * __restrict__ q, double * scalars, uint64_t n ) {
				const uint64_t i = static_cast< uint64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const double rho = scalars[ S_RHO ];
				const double alpha = __ddiv_rn( rho, scalars[ S_PQ ] ); // cg.hpp:127
				if( i < n ) {
					x[ i ] = __dadd_rn( __dmul_rn( 1.0, x[ i ] ), __dmul_rn( alpha, p[ i ] ) );  // cg.hpp:128
					r[ i ] = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -alpha, q[ i ] ) ); // cg.hpp:129
				}
				if( i == 0 ) {
					scalars[ S_RHO_PREV ] = rho; // cg.hpp:130 (nobody reads rho_prev in this launch)
				}
			}

			__global__ void k_cg_record( const double * __restrict__ scalars, double * hist_rr, double * hist_pq,
				unsigned int * iter_counter ) {
				const unsigned int it = *iter_counter;
				hist_rr[ it ] = scalars[ S_RR ];
				hist_pq[ it ] = scalars[ S_PQ ];
				*iter_counter = it + 1;
			}

			// ------------------------------------------------------------ setup kernels

			__device__ __forceinline__ int span( int i, int n ) {
				return ( i > 0 ? 1 : 0 ) + 1 + ( i + 1 < n ? 1 : 0 );
			}

			__global__ void k_stencil_widths( int nx, int ny, int nz, const int32_t * __restrict__ rows, int64_t npos,
				int64_t nslices, int32_t * __restrict__ widths ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( ( pos >> 5 ) >= nslices ) {
					return;
				}
				int count = 0;
				if( pos < npos ) {
					const int64_t i = rows ? rows[ pos ] : pos;
					if( i >= 0 ) {
						const int ix = static_cast< int >( i % nx );
						const int iy = static_cast< int >( ( i / nx ) % ny );
						const int iz = static_cast< int >( i / ( static_cast< int64_t >( nx ) * ny ) );
						count = span( ix, nx ) * span( iy, ny ) * span( iz, nz );
					}
				}
				const int width = __reduce_max_sync( 0xffffffffu, count );
				if( ( threadIdx.x & 31 ) == 0 ) {
					widths[ pos >> 5 ] = width;
				}
			}

			// problem.hpp:108-127: neighbours ascend lexicographically in (z,y,x), 26 on the
			// diagonal and -1 off it; remaining slots of the slice are padding (col -1).
			__global__ void k_stencil_fill( int nx, int ny, int nz, const int32_t * __restrict__ rows, int64_t npos,
				int64_t nslices, const int64_t * __restrict__ slice_off, double * __restrict__ vals,
				int32_t * __restrict__ cols ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const int64_t s = pos >> 5;
				if( s >= nslices ) {
					return;
				}
				int64_t e = slice_off[ s ] + ( pos & 31 );
				const int64_t end = slice_off[ s + 1 ];
				const int64_t i = pos < npos ? ( rows ? rows[ pos ] : pos ) : -1;
				if( i >= 0 ) {
					const int ix = static_cast< int >( i % nx );
					const int iy = static_cast< int >( ( i / nx ) % ny );
					const int iz = static_cast< int >( i / ( static_cast< int64_t >( nx ) * ny ) );
					for( int jz = iz > 0 ? iz - 1 : 0; jz < nz && jz <= iz + 1; ++jz ) {
						for( int jy = iy > 0 ? iy - 1 : 0; jy < ny && jy <= iy + 1; ++jy ) {
							for( int jx = ix > 0 ? ix - 1 : 0; jx < nx && jx <= ix + 1; ++jx ) {
								const int64_t j = jx + static_cast< int64_t >( nx ) * ( jy + static_cast< int64_t >( ny ) * jz );
								vals[ e ] = j == i ? 26.0 : -1.0;
								cols[ e ] = static_cast< int32_t >( j );
								e += kSlice;
							}
						}
					}
				}
				for( ; e < end; e += kSlice ) {
					vals[ e ] = 0.0;
					cols[ e ] = -1;
				}
			}

			__global__ void k_color_rows( int nx, int ny, int px, int py, int pz, int sx, int sy, int64_t pos0, int64_t size,
				int64_t padded, int32_t * __restrict__ rows ) {
				const int64_t q = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( q >= padded ) {
					return;
				}
				int32_t out = -1;
				if( q < size ) {
					const int cx = static_cast< int >( q % sx );
					const int cy = static_cast< int >( ( q / sx ) % sy );
					const int cz = static_cast< int >( q / ( static_cast< int64_t >( sx ) * sy ) );
					out = static_cast< int32_t >( ( 2 * cx + px )
						+ static_cast< int64_t >( nx ) * ( ( 2 * cy + py ) + static_cast< int64_t >( ny ) * ( 2 * cz + pz ) ) );
				}
				rows[ pos0 + q ] = out;
			}

			__global__ void k_injection_cols( int nx, int ny, int cxn, int cyn, int64_t nc, int32_t * __restrict__ fine ) {
				const int64_t c = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( c >= nc ) {
					return;
				}
				const int cx = static_cast< int >( c % cxn );
				const int cy = static_cast< int >( ( c / cxn ) % cyn );
				const int cz = static_cast< int >( c / ( static_cast< int64_t >( cxn ) * cyn ) );
				fine[ c ] = static_cast< int32_t >( 2 * cx + static_cast< int64_t >( nx ) * ( 2 * cy + static_cast< int64_t >( ny ) * 2 * cz ) );
			}

			__global__ void k_sell_single_entry( const int32_t * __restrict__ col_of_row, int64_t nrows, int64_t nslices,
				double * __restrict__ vals, int32_t * __restrict__ cols ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( ( pos >> 5 ) >= nslices ) {
					return;
				}
				const bool live = pos < nrows;
				vals[ pos ] = live ? 1.0 : 0.0;
				cols[ pos ] = live ? col_of_row[ pos ] : -1;
			}

			__global__ void k_sell_row_counts( const int64_t * __restrict__ slice_off, const int32_t * __restrict__ cols,
				int64_t nrows, int64_t * __restrict__ counts ) {
				const int64_t row = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( row >= nrows ) {
					return;
				}
				const int64_t s = row >> 5;
				int64_t count = 0;
				for( int64_t e = slice_off[ s ] + ( row & 31 ); e < slice_off[ s + 1 ]; e += kSlice ) {
					count += cols[ e ] >= 0 ? 1 : 0;
				}
				counts[ row ] = count;
			}

			__global__ void k_sell_to_csr( const int64_t * __restrict__ slice_off, const double * __restrict__ vals,
				const int32_t * __restrict__ cols, int64_t nrows, const int64_t * __restrict__ row_off,
				int64_t * __restrict__ out_cols, double * __restrict__ out_vals ) {
				const int64_t row = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( row >= nrows ) {
					return;
				}
				const int64_t s = row >> 5;
				int64_t at = row_off[ row ];
				for( int64_t e = slice_off[ s ] + ( row & 31 ); e < slice_off[ s + 1 ]; e += kSlice ) {
					if( cols[ e ] >= 0 ) {
						out_cols[ at ] = cols[ e ];
						out_vals[ at ] = vals[ e ];
						++at;
					}
				}
			}

		} // namespace

		// ================================================================ wrappers

		void fill( cudaStream_t st, double * v, uint64_t n, double value ) {
			if( n == 0 ) {
				return;
			}
			k_fill<<< blocks_for( n ), kBlock, 0, st >>>( v, n, value );
			count_launch();
		}

		void waxpby( cudaStream_t st, double * w, double alpha, const double * x, double beta, const double * y,
			uint64_t n ) {
			if( n == 0 ) {
				return;
			}
			k_waxpby<<< blocks_for( n ), kBlock, 0, st >>>( w, alpha, x, beta, y, n );
			count_launch();
		}

		void dot_exact( cudaStream_t st, const double * x, const double * y, uint64_t n, double * partials,
			unsigned int * counter, double * out ) {
			if( n == 0 ) {
				k_dot_empty<<< 1, 1, 0, st >>>( out );
				count_launch();
				return;
			}
			const unsigned int nchunks = static_cast< unsigned int >( ( n + kDotChunk - 1 ) / kDotChunk );
			k_dot_exact<<< nchunks, 32, 0, st >>>( x, y, n, partials, counter, out );
			count_launch();
		}

		uint64_t dot_tree_blocks( uint64_t n, int sm_count ) {
			const uint64_t want = ( n + kBlock * 8 - 1 ) / ( kBlock * 8 );
			const uint64_t cap = static_cast< uint64_t >( sm_count ) * 4;
			const uint64_t blocks = want < cap ? want : cap;
			return blocks < 1 ? 1 : blocks;
		}

		void dot_tree( cudaStream_t st, const double * x, const double * y, uint64_t n, int sm_count, double * partials,
			unsigned int * counter, double * out ) {
			if( n == 0 ) {
				k_dot_empty<<< 1, 1, 0, st >>>( out );
				count_launch();
				return;
			}
			const unsigned int blocks = static_cast< unsigned int >( dot_tree_blocks( n, sm_count ) );
			k_dot_tree<<< blocks, kBlock, 0, st >>>( x, y, n, partials, counter, out );
			count_launch();
		}

		void spmv( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			const double * x, double * y, int64_t nrows ) {
			if( nrows == 0 ) {
				return;
			}
			k_spmv<<< blocks_for( nrows ), kBlock, 0, st >>>( slice_off, vals, cols, x, y, nrows );
			count_launch();
		}

		void spmv_masked( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			const double * x, double * y, const int32_t * members, int64_t count ) {
			if( count == 0 ) {
				return;
			}
			k_spmv_masked<<< blocks_for( count ), kBlock, 0, st >>>( slice_off, vals, cols, x, y, members, count );
			count_launch();
		}

		void gs_color_step( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			const int32_t * rows, int64_t pos_begin, int64_t pos_count, double * z, const double * r ) {
			if( pos_count == 0 ) {
				return;
			}
			k_gs_color<<< blocks_for( pos_count ), kBlock, 0, st >>>( slice_off, vals, cols, rows, pos_begin, pos_count, z,
				r );
			count_launch();
		}

		void residual_restrict( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			const int32_t * rows, int64_t n_coarse, const double * z, const double * r, double * r_c ) {
			if( n_coarse == 0 ) {
				return;
			}
			k_residual_restrict<<< blocks_for( n_coarse ), kBlock, 0, st >>>( slice_off, vals, cols, rows, n_coarse, z, r,
				r_c );
			count_launch();
		}

		void prolong_add( cudaStream_t st, const int32_t * rows, int64_t n_coarse, double * z, const double * z_c ) {
			if( n_coarse == 0 ) {
				return;
			}
			k_prolong_add<<< blocks_for( n_coarse ), kBlock, 0, st >>>( rows, n_coarse, z, z_c );
			count_launch();
		}

		void cg_update_p( cudaStream_t st, double * p, const double * z, const double * scalars,
			const unsigned int * iter_counter, uint64_t n ) {
			if( n == 0 ) {
				return;
			}
			k_cg_update_p<<< blocks_for( n ), kBlock, 0, st >>>( p, z, scalars, iter_counter, n );
			count_launch();
		}

		void cg_update_xr( cudaStream_t st, double * x, double * r, const double * p, const double * q, double * scalars,
			uint64_t n ) {
			k_cg_update_xr<<< n == 0 ? 1 : blocks_for( n ), kBlock, 0, st >>>( x, r, p, q, scalars, n );
			count_launch();
		}

		void cg_record( cudaStream_t st, const double * scalars, double * hist_rr, double * hist_pq,
			unsigned int * iter_counter ) {
			k_cg_record<<< 1, 1, 0, st >>>( scalars, hist_rr, hist_pq, iter_counter );
			count_launch();
		}

		void stencil_widths( cudaStream_t st, int nx, int ny, int nz, const int32_t * rows, int64_t npos, int64_t nslices,
			int32_t * widths ) {
			if( nslices == 0 ) {
				return;
			}
			k_stencil_widths<<< blocks_for( nslices * kSlice ), kBlock, 0, st >>>( nx, ny, nz, rows, npos, nslices, widths );
			count_launch();
		}

		void stencil_fill( cudaStream_t st, int nx, int ny, int nz, const int32_t * rows, int64_t npos, int64_t nslices,
			const int64_t * slice_off, double * vals, int32_t * cols ) {
			if( nslices == 0 ) {
				return;
			}
			k_stencil_fill<<< blocks_for( nslices * kSlice ), kBlock, 0, st >>>( nx, ny, nz, rows, npos, nslices, slice_off,
				vals, cols );
			count_launch();
		}

		void color_rows( cudaStream_t st, int nx, int ny, int nz, int px, int py, int pz, int64_t pos0, int64_t size,
			int64_t padded, int32_t * rows ) {
			(void) nz;
			if( padded == 0 ) {
				return;
			}
			const int sx = ( nx + 1 - px ) / 2;
			const int sy = ( ny + 1 - py ) / 2;
			k_color_rows<<< blocks_for( padded ), kBlock, 0, st >>>( nx, ny, px, py, pz, sx > 0 ? sx : 1, sy > 0 ? sy : 1,
				pos0, size, padded, rows );
			count_launch();
		}

		void injection_cols( cudaStream_t st, int nx, int ny, int nz, int32_t * fine ) {
			const int64_t nc = static_cast< int64_t >( nx / 2 ) * ( ny / 2 ) * ( nz / 2 );
			if( nc == 0 ) {
				return;
			}
			k_injection_cols<<< blocks_for( nc ), kBlock, 0, st >>>( nx, ny, nx / 2, ny / 2, nc, fine );
			count_launch();
		}

		void sell_single_entry( cudaStream_t st, const int32_t * col_of_row, int64_t nrows, int64_t nslices, double * vals,
			int32_t * cols ) {
			if( nslices == 0 ) {
				return;
			}
			k_sell_single_entry<<< blocks_for( nslices * kSlice ), kBlock, 0, st >>>( col_of_row, nrows, nslices, vals,
				cols );
			count_launch();
		}

		void sell_row_counts( cudaStream_t st, const int64_t * slice_off, const int32_t * cols, int64_t nrows,
			int64_t * counts ) {
			if( nrows == 0 ) {
				return;
			}
			k_sell_row_counts<<< blocks_for( nrows ), kBlock, 0, st >>>( slice_off, cols, nrows, counts );
			count_launch();
		}

		void sell_to_csr( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			int64_t nrows, const int64_t * row_off, int64_t * out_cols, double * out_vals ) {
			if( nrows == 0 ) {
				return;
			}
			k_sell_to_csr<<< blocks_for( nrows ), kBlock, 0, st >>>( slice_off, vals, cols, nrows, row_off, out_cols,
				out_vals );
			count_launch();
		}

	} // namespace kern
} // namespace slabgpu
