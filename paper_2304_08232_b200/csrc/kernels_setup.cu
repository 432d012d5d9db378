// kernels_setup.cu — setup-time kernels: the 27-point stencil generated straight into SELL-32
// (problem.hpp:90-131) for the box a rank owns (the whole grid on one GPU), colour row lists, the
// injection restriction (problem.hpp:174-201) and the SELL -> CSR download path. None of these
// run inside a solve.
#include "kernels.cuh"

#include <cuda_runtime.h>

#include "common.hpp"
#include "decomp.hpp"

namespace slabgpu {
	namespace kern {

		namespace {

			constexpr int kBlock = 256;

			inline unsigned int blocks_for( uint64_t count, int block = kBlock ) {
				return static_cast< unsigned int >( ( count + block - 1 ) / block );
			}

			// owned row -> global coordinates
			__device__ __forceinline__ void row_coords( const Decomp & D, int64_t i, int & X, int & Y, int & Z ) {
				const int ix = static_cast< int >( i % D.l[ 0 ] );
				const int iy = static_cast< int >( ( i / D.l[ 0 ] ) % D.l[ 1 ] );
				const int iz = static_cast< int >( i / ( static_cast< int64_t >( D.l[ 0 ] ) * D.l[ 1 ] ) );
				X = D.o[ 0 ] + ix;
				Y = D.o[ 1 ] + iy;
				Z = D.o[ 2 ] + iz;
			}

			__global__ void k_stencil_widths( const Decomp D, const int32_t * __restrict__ rows, int64_t npos,
				int64_t nslices, int32_t * __restrict__ widths ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( ( pos >> 5 ) >= nslices ) {
					return;
				}
				int count = 0;
				if( pos < npos ) {
					const int64_t i = rows ? rows[ pos ] : pos;
					if( i >= 0 ) {
						int X, Y, Z;
						row_coords( D, i, X, Y, Z );
						count = span_1d( X, D.g[ 0 ] ) * span_1d( Y, D.g[ 1 ] ) * span_1d( Z, D.g[ 2 ] );
					}
				}
				const int width = __reduce_max_sync( 0xffffffffu, count );
				if( ( threadIdx.x & 31 ) == 0 ) {
					widths[ pos >> 5 ] = width;
				}
			}

			// problem.hpp:108-127: neighbours ascend lexicographically in (z,y,x) of the GLOBAL grid,
			// 26 on the diagonal and -1 off it; columns are local indices (owned or ghost);
			// remaining slots of the slice are padding (col -1).
			__global__ void k_stencil_fill( const Decomp D, const int32_t * __restrict__ rows, int64_t npos,
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
					int X, Y, Z;
					row_coords( D, i, X, Y, Z );
					for( int jz = Z > 0 ? Z - 1 : 0; jz < D.g[ 2 ] && jz <= Z + 1; ++jz ) {
						for( int jy = Y > 0 ? Y - 1 : 0; jy < D.g[ 1 ] && jy <= Y + 1; ++jy ) {
							for( int jx = X > 0 ? X - 1 : 0; jx < D.g[ 0 ] && jx <= X + 1; ++jx ) {
								const bool diagonal = jx == X && jy == Y && jz == Z;
								vals[ e ] = diagonal ? 26.0 : -1.0;
								cols[ e ] = local_index( D, jx, jy, jz );
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

			// members of global parity class (cx,cy,cz) inside the owned box, ascending local index
			__global__ void k_color_rows( const Decomp D, int cx, int cy, int cz, int64_t pos0, int64_t size, int64_t padded,
				int32_t * __restrict__ rows ) {
				const int64_t q = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( q >= padded ) {
					return;
				}
				int32_t out = -1;
				if( q < size ) {
					const int sx = count_parity( D.o[ 0 ], D.l[ 0 ], cx );
					const int sy = count_parity( D.o[ 1 ], D.l[ 1 ], cy );
					const int qx = static_cast< int >( q % sx );
					const int qy = static_cast< int >( ( q / sx ) % sy );
					const int qz = static_cast< int >( q / ( static_cast< int64_t >( sx ) * sy ) );
					const int ix = first_parity( D.o[ 0 ], cx ) - D.o[ 0 ] + 2 * qx;
					const int iy = first_parity( D.o[ 1 ], cy ) - D.o[ 1 ] + 2 * qy;
					const int iz = first_parity( D.o[ 2 ], cz ) - D.o[ 2 ] + 2 * qz;
					out = static_cast< int32_t >( ix + static_cast< int64_t >( D.l[ 0 ] ) * ( iy + static_cast< int64_t >( D.l[ 1 ] ) * iz ) );
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

			// halo pack: buf[dst[k]] = v[src[k]]  (dst == nullptr: buf[k])
			__global__ void k_halo_pack( const int32_t * __restrict__ src, const int32_t * __restrict__ dst, int64_t count,
				const double * __restrict__ v, double * __restrict__ buf ) {
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( k < count ) {
					buf[ dst != nullptr ? dst[ k ] : k ] = v[ src[ k ] ];
				}
			}

		} // namespace

		void stencil_widths( cudaStream_t st, const Decomp & D, const int32_t * rows, int64_t npos, int64_t nslices,
			int32_t * widths ) {
			if( nslices == 0 ) {
				return;
			}
			k_stencil_widths<<< blocks_for( nslices * kSlice ), kBlock, 0, st >>>( D, rows, npos, nslices, widths );
			count_launch();
		}

		void stencil_fill( cudaStream_t st, const Decomp & D, const int32_t * rows, int64_t npos, int64_t nslices,
			const int64_t * slice_off, double * vals, int32_t * cols ) {
			if( nslices == 0 ) {
				return;
			}
			k_stencil_fill<<< blocks_for( nslices * kSlice ), kBlock, 0, st >>>( D, rows, npos, nslices, slice_off, vals,
				cols );
			count_launch();
		}

		void color_rows( cudaStream_t st, const Decomp & D, int color, int64_t pos0, int64_t size, int64_t padded,
			int32_t * rows ) {
			if( padded == 0 ) {
				return;
			}
			k_color_rows<<< blocks_for( padded ), kBlock, 0, st >>>( D, color & 1, ( color >> 1 ) & 1, ( color >> 2 ) & 1, pos0,
				size, padded, rows );
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

		void halo_pack( cudaStream_t st, const int32_t * src, const int32_t * dst, int64_t count, const double * v,
			double * buf ) {
			if( count == 0 ) {
				return;
			}
			k_halo_pack<<< blocks_for( count ), kBlock, 0, st >>>( src, dst, count, v, buf );
			count_launch();
		}

	} // namespace kern
} // namespace slabgpu
