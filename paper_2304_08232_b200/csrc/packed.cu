// packed.cu — dictionary-coded SELL: the matrix stream of the hot kernels cut from 12 bytes to 1 byte
// per stored entry, with results that are bit-identical to the plain format.
//
// Why. Every product and colour step of the solve is bound by the matrix stream (12 B per entry against
// 8 B per row of vector traffic). A matrix handed to the library is immutable and opaque
// (sparse_matrix.hpp:48-171), so its device copy may be any lossless encoding. Matrices that come from
// a discretisation repeat very few distinct (column - row, value) pairs — the 27-point operator of this
// benchmark has 27 — so each entry is stored as the 8-bit index of its pair in a per-matrix dictionary
// that is discovered from the entries themselves (no knowledge of where the matrix came from). The
// decode is exact: the value is the dictionary's double, the column is row + delta in integers, and the
// entries of a row are visited in the same ascending-column order (operations.hpp:116-125). Rows with
// an entry outside the dictionary (ghost columns of a decomposed level, irregular matrices) are
// flagged and read from the plain arrays by the same thread. Matrices that do not compress keep the
// plain kernels.
//
// With the stream 12x smaller, a fine-level colour step stops evicting the vector it gathers from the
// L2; what bounds the kernels then is the L1 request path of the gathers, so everything else is kept off
// it and the decode is a handful of instructions per entry: value and offset come from the dictionary
// through indexed constant loads (the dictionary is a kernel parameter), full rows (no padding inside
// the width class) skip the per-entry padding test, the diagonal a colour step divides by is named by a
// spare byte of the row instead of being searched for, and many-wave launches give a thread several
// rows that share their codes.
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>
#include <type_traits>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"
#include "packed_decode.cuh"

namespace slabgpu {

	int g_use_packed = 1;
	int g_pack_build = 1;
	// keep the plain SELL arrays of a matrix whose coded copy has no escaped rows? 0 frees them (324 -> 32 bytes
	// per 27-point row, i.e. 4-5x larger grids per GPU); such a matrix always runs the coded kernels and can no
	// longer be downloaded or transposed. Set before the matrix is created.
	int g_keep_plain = 1;
	int g_packed_block = 256;
	// Tuning, all measured on B200 (tools/kernel_microbench.py, tools/solve_sweep.py):
	// single-row kernels gather two 4-code words at a time (the launches they serve, 65k-300k rows, are
	// latency-bound; one word at a time is better only for many-wave launches, which the multi-row kernels
	// take; the whole row at once was never better once the dictionary left shared memory)
	int g_packed_batch = 2;
	int g_packed_rows = 2;               // rows per thread where rows repeat their codes at a fixed distance (1 = off):
	int g_packed_rows_spmv = 3;          // ... colour steps / products (measured on B200, tools/kernel_microbench.py)
	int64_t g_packed_multi_min_rows = 300000; // ... for launches of at least this many rows
	int64_t g_packed_min_rows = 65536;   // launches below this many rows use the plain kernels (measured: their
	                                     // matrices sit in the L2, where the plain preload shape is faster)

	void Packed::release() {
		if( codes ) cudaFree( codes );
		if( dict ) cudaFree( dict );
		delete[] h_dict;
		codes = nullptr;
		dict = nullptr;
		h_dict = nullptr;
		max_width = ncodes = chunks = dict_size = stride = 0;
		escaped_rows = 0;
	}

	namespace kern {

		namespace {

			using namespace dev;
			using namespace coded;

// the two-rows-per-thread colour step at 4 resident blocks per SM (64 registers): +4 % over the
// compiler's own 70; 5 blocks spill and lose 15 % (measured at 192^3)
#ifndef GS_MULTI_MINBLOCKS
#define GS_MULTI_MINBLOCKS 4
#endif
			constexpr int kDict = 256;
			constexpr int kMaxCodes = 64;
			constexpr int kMaxChunks = ( kMaxCodes + 16 ) / 16;

			// width classes the kernels are instantiated for
			int width_class( int max_width ) {
				const int classes[] = { 8, 16, 27, 32, 64 };
				for( int c : classes ) {
					if( max_width <= c ) {
						return c;
					}
				}
				return 0;
			}

			// ------------------------------------------------------------ encoder (setup)

			// one thread per row position: looks every entry up in the dictionary and writes the row's
			// codes; entries that are missing flag the row and are offered as candidates
			__global__ void __launch_bounds__( kBlock ) k_pack_rows( const int64_t * __restrict__ slice_off,
				const double * __restrict__ vals, const int32_t * __restrict__ cols, const int32_t * __restrict__ rows,
				int64_t npos, int64_t npadded, const DictEntry * __restrict__ dict, int dict_size, int chunks,
				uint4 * __restrict__ codes, unsigned long long * escaped, unsigned long long * cand_key, unsigned int cand_cap,
				double * cand_val, int32_t * cand_delta, unsigned int * cand_hits, int32_t owned_cols ) {
				__shared__ long long s_val[ kDict ];
				__shared__ int32_t s_delta[ kDict ];
				for( int t = threadIdx.x; t < dict_size; t += blockDim.x ) {
					s_val[ t ] = __double_as_longlong( dict[ t ].val );
					s_delta[ t ] = dict[ t ].delta;
				}
				__syncthreads();
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( pos >= npadded ) {
					return;
				}
				const int64_t s = pos >> 5;
				const int lane = static_cast< int >( pos & 31 );
				const int64_t row = pos < npos ? ( rows != nullptr ? static_cast< int64_t >( rows[ pos ] ) : pos ) : -1;
				unsigned int w[ 4 * kMaxChunks ];
				#pragma unroll
				for( int j = 0; j < 4 * kMaxChunks; ++j ) {
					w[ j ] = 0u;
				}
				bool escape = false;
				unsigned int diag_code = 0u;
				if( row >= 0 ) {
					const int64_t base = slice_off[ s ];
					const int width = static_cast< int >( ( slice_off[ s + 1 ] - base ) >> 5 );
					for( int k = 0; k < width; ++k ) {
						const int64_t e = base + static_cast< int64_t >( k ) * kSlice + lane;
						const int32_t c = cols[ e ];
						if( c < 0 ) {
							continue; // padding keeps code 0
						}
						const long long bits = __double_as_longlong( vals[ e ] );
						const int32_t delta = c - static_cast< int32_t >( row );
						unsigned int code = 0u;
						for( int t = 1; t < dict_size; ++t ) {
							if( s_delta[ t ] == delta && s_val[ t ] == bits ) {
								code = static_cast< unsigned int >( t );
								break;
							}
						}
						if( delta == 0 ) {
							diag_code = code;
						}
						if( code == 0u ) {
							escape = true;
						}
						// columns beyond the owned ones are ghost slots of a decomposed level: their offsets repeat
						// nowhere, so they are never offered (they would only crowd the regular pairs out of the set)
						if( code == 0u && c < owned_cols ) {
							// offer the pair: open-addressing set keyed by a 64-bit mix of the pair. (Two different
							// pairs with one key are vanishingly rare and only delay the second by a round.)
							unsigned long long key = ( static_cast< unsigned long long >( bits ) * 0x9E3779B97F4A7C15ull )
								^ ( static_cast< unsigned long long >( static_cast< uint32_t >( delta ) ) * 0xC2B2AE3D27D4EB4Full );
							key |= 1ull;
							unsigned int slot = static_cast< unsigned int >( ( key >> 20 ) % cand_cap );
							bool listed = false;
							for( unsigned int probe = 0; probe < 64u && !listed; ++probe ) {
								const unsigned long long cur = reinterpret_cast< volatile unsigned long long * >( cand_key )[ slot ];
								if( cur == key ) {
									listed = true;
								} else if( cur == 0ull ) {
									const unsigned long long old = atomicCAS( cand_key + slot, 0ull, key );
									if( old == 0ull ) {
										cand_val[ slot ] = vals[ e ];
										cand_delta[ slot ] = delta;
									}
									listed = old == 0ull || old == key;
								}
								if( !listed ) {
									slot = slot + 1 == cand_cap ? 0u : slot + 1;
								}
							}
							// how common is the pair? counted on every 64th row: the dictionary takes the most frequent
							// pairs first (the ghost columns of a decomposed level offer thousands of pairs that occur once)
							if( listed && ( pos & 63 ) == 0 ) {
								atomicAdd( cand_hits + slot, 1u );
							}
						}
						#pragma unroll
						for( int j = 0; j < 4 * kMaxChunks; ++j ) { // static indexing keeps w in registers
							if( j == ( k >> 2 ) ) {
								w[ j ] |= code << ( 8 * ( k & 3 ) );
							}
						}
					}
				}
				if( escape ) {
					w[ 0 ] = ( w[ 0 ] & ~0xffu ) | kEscape;
					atomicAdd( escaped, 1ull );
				}
				#pragma unroll
				for( int j = 0; j < 4 * kMaxChunks; ++j ) { // the row's last byte names its diagonal entry
					if( j == 4 * chunks - 1 ) {
						w[ j ] |= diag_code << 24;
					}
				}
				#pragma unroll
				for( int j = 0; j < kMaxChunks; ++j ) {
					if( j < chunks ) {
						codes[ ( s * chunks + j ) * kSlice + lane ] = make_uint4( w[ 4 * j ], w[ 4 * j + 1 ], w[ 4 * j + 2 ], w[ 4 * j + 3 ] );
					}
				}
			}

			// (decoder: packed_decode.cuh)


			// ------------------------------------------------------------ kernels

			// operations.hpp:164-174; MASKED: one thread per mask member, others untouched.
			// (x and y deliberately without __restrict__: ordinary loads obey the scheduling fence in coded_row_sum)
			template< int NCODES, int CHUNKS, int BATCH, bool MASKED, int DICT >
			__global__ void __launch_bounds__( kBlock ) k_spmv_packed( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const double * x, double * y,
				const int32_t * __restrict__ members, int64_t count, double * dot_partials ) {
				__shared__ double smem[ 32 ];
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const bool live = k < count;
				int64_t row = 0;
				RowCodes< CHUNKS > rc;
				if( live ) {
					row = MASKED ? members[ k ] : k;
					codes_load( codes, row, rc );
				}
				dep_trigger();
				dep_wait();
				double prod = 0.0;
				if( live ) {
					const bool warp_ragged = __any_sync( __activemask(), rc.template ragged< NCODES >() );
					double unused = 0.0;
					const double acc = any_row_sum< NCODES, CHUNKS, BATCH, false >( rc, warp_ragged, plain, row, static_cast< int32_t >( row ), x, dp, unused );
					y[ row ] = acc;
					prod = dot_partials != nullptr ? __dmul_rn( x[ row ], acc ) : 0.0;
				}
				if( dot_partials != nullptr ) { // x'(A x): block partials, folded by sum_partials (cg.hpp:122-123)
					const double block_sum = block_tree_sum( prod, smem );
					if( threadIdx.x == 0 ) {
						dot_partials[ blockIdx.x ] = block_sum;
					}
				}
			}

			// smoother.hpp:60-72 fused, with the grid transfers of kernels.cu's k_gs_color riding on the
			// colour-0 steps (flags bit 0: prolongation in front, bit 1: residual + restriction behind)
			template< int NCODES, int CHUNKS, int BATCH, int DICT >
			__global__ void __launch_bounds__( kBlock, 4 ) k_gs_color_packed( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows,
				int64_t pos_begin, int64_t pos_count, double * z, const double * r, int flags,
				const double * src, double * out, double * zero,
				const int32_t * __restrict__ pos_list, const uint8_t * __restrict__ skip ) {
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				int32_t i = -1;
				int64_t pos = 0;
				RowCodes< CHUNKS > rc;
				if( k < pos_count ) {
					pos = pos_list != nullptr ? pos_list[ k ] : pos_begin + k;
					// rows == nullptr: vectors in position order (row index == position)
					i = skip != nullptr && skip[ pos ] ? -1 : ( rows != nullptr ? rows[ pos ] : static_cast< int32_t >( pos ) );
					codes_load( codes, pos, rc );
				}
				dep_trigger();
				dep_wait();
				if( i < 0 ) {
					return;
				}
				const bool warp_ragged = __any_sync( __activemask(), rc.template ragged< NCODES >() );
				const int64_t coarse = pos - pos_begin;
				const double ri = r[ i ];
				double zi = z[ i ];
				if( flags & 1 ) {
					const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ coarse ] ) );
					zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
					z[ i ] = zi;
				}
				// flags bit 2: the step runs twice in a row (the last colour of a forward sweep is the first of the
				// backward sweep, smoother.hpp:108-111); nothing but z[i] itself changes in between
				const int passes = ( flags & 4 ) ? 2 : 1;
				#pragma unroll 1
				for( int pass = 0; pass < passes; ++pass ) {
					double d = 0.0;
					const double s = any_row_sum< NCODES, CHUNKS, BATCH, true >( rc, warp_ragged, plain, pos, i, z, dp, d );
					zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -s ), __dmul_rn( zi, d ) ), d );
					z[ i ] = zi;
				}
				if( flags & 2 ) {
					double unused = 0.0;
					const double az = any_row_sum< NCODES, CHUNKS, BATCH, false >( rc, warp_ragged, plain, pos, i, z, dp, unused );
					const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
					out[ coarse ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
					zero[ coarse ] = 0.0;
				}
			}

			// multigrid.hpp:100-104 on the injected rows (the colour-0 block): r_c[p] = 0 + 1*(1*r[i] + (-1)*(A z)[i])
			template< int NCODES, int CHUNKS, int BATCH, int DICT >
			__global__ void __launch_bounds__( kBlock ) k_residual_restrict_packed( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows,
				int64_t n_coarse, const double * z, const double * r, double * r_c, double * zero ) {
				const int64_t p = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const bool live = p < n_coarse;
				int32_t i = 0;
				RowCodes< CHUNKS > rc;
				if( live ) {
					i = rows[ p ];
					codes_load( codes, p, rc );
				}
				dep_trigger();
				dep_wait();
				if( !live ) {
					return;
				}
				const bool warp_ragged = __any_sync( __activemask(), rc.template ragged< NCODES >() );
				double unused = 0.0;
				const double az = any_row_sum< NCODES, CHUNKS, BATCH, false >( rc, warp_ragged, plain, p, i, z, dp, unused );
				const double f = __dadd_rn( __dmul_rn( 1.0, r[ i ] ), __dmul_rn( -1.0, az ) );
				r_c[ p ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
				if( zero != nullptr ) {
					zero[ p ] = 0.0; // set_all(z_c, 0), multigrid.hpp:104
				}
			}

			// ------------------------------------------------------------ several rows per thread

			// Rows that lie a fixed number of slices apart mostly carry the same codes (same place in the
			// next grid line). A thread that owns R such rows decodes every code once and applies it to all
			// of them: R times fewer constant-cache reads and decode instructions, R times more gathers in
			// flight per thread, and the R rows re-read each other's neighbourhood while it is still in L1.
			// The arithmetic of each row and its order are unchanged.
			template< int CHUNKS >
			__device__ __forceinline__ bool same_codes( const RowCodes< CHUNKS > & a, const RowCodes< CHUNKS > & b ) {
				unsigned int diff = 0u;
				#pragma unroll
				for( int j = 0; j < CHUNKS; ++j ) {
					diff |= ( a.q[ j ].x ^ b.q[ j ].x ) | ( a.q[ j ].y ^ b.q[ j ].y ) | ( a.q[ j ].z ^ b.q[ j ].z ) | ( a.q[ j ].w ^ b.q[ j ].w );
				}
				return diff == 0u;
			}

			template< int NCODES, int CHUNKS, int R, bool RAGGED, int DICT >
			__device__ __forceinline__ void shared_rows_sum( const RowCodes< CHUNKS > & rc, const double * x, const int32_t ( &row )[ R ],
				const DictParam< DICT > & dp, double ( &acc )[ R ] ) {
				// (row + delta in 32 bits, then one widening multiply-add per gather: with per-row pointers the
				//  compiler rebuilds each 64-bit address from the row index, five instructions per gather)
				constexpr int WORDS = ( NCODES + 3 ) / 4;
				#pragma unroll
				for( int r = 0; r < R; ++r ) {
					acc[ r ] = 0.0;
				}
				#pragma unroll
				for( int wi = 0; wi < WORDS; ++wi ) {
					const unsigned int word = rc.word( wi );
					double v[ 4 ], xv[ R ][ 4 ];
					int32_t dl[ 4 ];
					#pragma unroll
					for( int j = 0; j < 4; ++j ) {
						if( 4 * wi + j < NCODES ) {
							const unsigned int code = ( word >> ( 8 * j ) ) & 0xffu;
							dl[ j ] = dp.e[ code ].delta;
							v[ j ] = dp.e[ code ].val;
						}
					}
					#pragma unroll
					for( int r = 0; r < R; ++r ) {
						#pragma unroll
						for( int j = 0; j < 4; ++j ) {
							if( 4 * wi + j < NCODES ) {
								xv[ r ][ j ] = x[ row[ r ] + dl[ j ] ];
							}
						}
					}
					#pragma unroll
					for( int r = 0; r < R; ++r ) {
						#pragma unroll
						for( int j = 0; j < 4; ++j ) {
							if( 4 * wi + j < NCODES ) {
								const double prod = __dmul_rn( v[ j ], xv[ r ][ j ] );
								if( !RAGGED || ( ( word >> ( 8 * j ) ) & 0xffu ) != 0u ) {
									acc[ r ] = __dadd_rn( acc[ r ], prod );
								}
							}
						}
					}
				}
			}

			// position of row r of this thread: warp `gw` of the launch owns lane-columns of the slices
			// first + tile*R*stride + j + r*stride, tile = gw / stride, j = gw % stride
			// (32-bit arithmetic: a 64-bit division is a ~100-instruction subroutine, and every thread would run it)
			template< int R >
			__device__ __forceinline__ int64_t multi_first_slice( int64_t first_slice, unsigned int gw, unsigned int stride ) {
				const unsigned int tile = gw / stride;
				const unsigned int j = gw - tile * stride;
				return first_slice + static_cast< int64_t >( tile ) * ( R * stride ) + j;
			}

			// k_gs_color_packed with R rows per thread; covers the contiguous range [pos_begin, pos_begin + pos_count)
			template< int NCODES, int CHUNKS, int R, int DICT >
			__global__ void __launch_bounds__( kBlock, R == 2 ? GS_MULTI_MINBLOCKS : ( R == 3 ? 3 : 2 ) ) k_gs_color_packed_multi( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows, int stride,
				int64_t pos_begin, int64_t pos_count, double * z, const double * r, int flags,
				const double * src, double * out, double * zero ) {
				const int lane = threadIdx.x & 31;
				const unsigned int gw = ( blockIdx.x * blockDim.x + threadIdx.x ) >> 5;
				const int64_t slice0 = multi_first_slice< R >( pos_begin >> 5, gw, static_cast< unsigned int >( stride ) );
				int32_t i[ R ];
				int64_t pos[ R ];
				RowCodes< CHUNKS > rc[ R ];
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					pos[ q ] = ( slice0 + static_cast< int64_t >( q ) * stride ) * kSlice + lane;
					i[ q ] = -1;
					#pragma unroll
					for( int j = 0; j < CHUNKS; ++j ) {
						rc[ q ].q[ j ] = make_uint4( 0u, 0u, 0u, 0u );
					}
					if( pos[ q ] < pos_begin + pos_count ) {
						i[ q ] = rows != nullptr ? rows[ pos[ q ] ] : static_cast< int32_t >( pos[ q ] );
						codes_load( codes, pos[ q ], rc[ q ] );
					}
				}
				dep_trigger();
				dep_wait();
				bool same = i[ 0 ] >= 0 && !rc[ 0 ].escaped();
				#pragma unroll
				for( int q = 1; q < R; ++q ) {
					same = same && i[ q ] >= 0 && same_codes( rc[ q ], rc[ 0 ] );
				}
				const bool shared = __all_sync( 0xffffffffu, same );
				const bool warp_ragged = __any_sync( 0xffffffffu, rc[ 0 ].template ragged< NCODES >() );
				if( shared ) {
					double ri[ R ], zi[ R ], acc[ R ];
					#pragma unroll
					for( int q = 0; q < R; ++q ) {
						ri[ q ] = r[ i[ q ] ];
						zi[ q ] = z[ i[ q ] ];
						if( flags & 1 ) {
							const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ pos[ q ] - pos_begin ] ) );
							zi[ q ] = __dadd_rn( __dmul_rn( 1.0, zi[ q ] ), __dmul_rn( 1.0, f ) );
							z[ i[ q ] ] = zi[ q ];
						}
					}
					const double d = dp.e[ rc[ 0 ].diag_code() ].val;
					const int passes = ( flags & 4 ) ? 2 : 1; // see k_gs_color_packed
					#pragma unroll 1
					for( int pass = 0; pass < passes; ++pass ) {
						if( warp_ragged ) {
							shared_rows_sum< NCODES, CHUNKS, R, true >( rc[ 0 ], z, i, dp, acc );
						} else {
							shared_rows_sum< NCODES, CHUNKS, R, false >( rc[ 0 ], z, i, dp, acc );
						}
						#pragma unroll
						for( int q = 0; q < R; ++q ) {
							zi[ q ] = __ddiv_rn( __dadd_rn( __dadd_rn( ri[ q ], -acc[ q ] ), __dmul_rn( zi[ q ], d ) ), d );
							z[ i[ q ] ] = zi[ q ];
						}
					}
					if( flags & 2 ) {
						if( warp_ragged ) {
							shared_rows_sum< NCODES, CHUNKS, R, true >( rc[ 0 ], z, i, dp, acc );
						} else {
							shared_rows_sum< NCODES, CHUNKS, R, false >( rc[ 0 ], z, i, dp, acc );
						}
						#pragma unroll
						for( int q = 0; q < R; ++q ) {
							const double f = __dadd_rn( __dmul_rn( 1.0, ri[ q ] ), __dmul_rn( -1.0, acc[ q ] ) );
							out[ pos[ q ] - pos_begin ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
							zero[ pos[ q ] - pos_begin ] = 0.0;
						}
					}
					return;
				}
				// rows that differ (grid boundaries, escaped rows, the tail of the range): one at a time
				// (unrolled: indexing the per-row arrays with a run-time q would push them to local memory)
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					if( i[ q ] < 0 ) {
						continue;
					}
					const int64_t coarse = pos[ q ] - pos_begin;
					const double ri = r[ i[ q ] ];
					double zi = z[ i[ q ] ];
					if( flags & 1 ) {
						const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ coarse ] ) );
						zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
						z[ i[ q ] ] = zi;
					}
					const int passes = ( flags & 4 ) ? 2 : 1;
					#pragma unroll 1
					for( int pass = 0; pass < passes; ++pass ) {
						double d = 0.0;
						const double sum = any_row_sum< NCODES, CHUNKS, 1, true >( rc[ q ], true, plain, pos[ q ], i[ q ], z, dp, d );
						zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -sum ), __dmul_rn( zi, d ) ), d );
						z[ i[ q ] ] = zi;
					}
					if( flags & 2 ) {
						double unused = 0.0;
						const double az = any_row_sum< NCODES, CHUNKS, 1, false >( rc[ q ], true, plain, pos[ q ], i[ q ], z, dp, unused );
						const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
						out[ coarse ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
						zero[ coarse ] = 0.0;
					}
				}
			}

			// k_gs_color_packed_multi for the interior launch of a colour on a decomposed level (skip flags)
			template< int NCODES, int CHUNKS, int R, int DICT >
			__global__ void __launch_bounds__( kBlock ) k_gs_color_packed_multi_skip( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows, int stride,
				int64_t pos_begin, int64_t pos_count, double * z, const double * r, int flags,
				const double * src, double * out, double * zero,
				const uint8_t * __restrict__ skip ) {
				// skip: positions flagged here are left out (the interior launch of a colour on a decomposed level,
				// whose boundary rows went first); such rows — like the padding at the end of the range — take part in
				// the shared decode as passengers: they borrow a live row's codes and address and store nothing
				const int lane = threadIdx.x & 31;
				const unsigned int gw = ( blockIdx.x * blockDim.x + threadIdx.x ) >> 5;
				const int64_t slice0 = multi_first_slice< R >( pos_begin >> 5, gw, static_cast< unsigned int >( stride ) );
				int32_t i[ R ];
				int64_t pos[ R ];
				RowCodes< CHUNKS > rc[ R ];
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					pos[ q ] = ( slice0 + static_cast< int64_t >( q ) * stride ) * kSlice + lane;
					i[ q ] = -1;
					#pragma unroll
					for( int j = 0; j < CHUNKS; ++j ) {
						rc[ q ].q[ j ] = make_uint4( 0u, 0u, 0u, 0u );
					}
					if( pos[ q ] < pos_begin + pos_count && !( skip != nullptr && skip[ pos[ q ] ] ) ) {
						i[ q ] = rows != nullptr ? rows[ pos[ q ] ] : static_cast< int32_t >( pos[ q ] );
						if( i[ q ] >= 0 ) {
							codes_load( codes, pos[ q ], rc[ q ] );
						}
					}
				}
				dep_trigger();
				dep_wait();
				// the lane's leader: its first live row (none: an idle lane with all-padding codes)
				int lead = -1;
				#pragma unroll
				for( int q = R - 1; q >= 0; --q ) {
					lead = i[ q ] >= 0 ? q : lead;
				}
				RowCodes< CHUNKS > lc = rc[ 0 ];
				int32_t li = 0;
				#pragma unroll
				for( int q = 1; q < R; ++q ) {
					if( lead == q ) {
						lc = rc[ q ];
					}
				}
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					li = lead == q ? i[ q ] : li;
				}
				bool same = lead < 0 || !lc.escaped();
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					same = same && ( i[ q ] < 0 || same_codes( rc[ q ], lc ) );
				}
				const bool shared = __all_sync( 0xffffffffu, same );
				const bool warp_ragged = __any_sync( 0xffffffffu, lc.template ragged< NCODES >() );
				if( shared ) {
					double ri[ R ], zi[ R ], acc[ R ];
					int32_t at[ R ];
					#pragma unroll
					for( int q = 0; q < R; ++q ) {
						at[ q ] = i[ q ] >= 0 ? i[ q ] : li; // passengers read the leader's row (row 0 on idle lanes)
						ri[ q ] = r[ at[ q ] ];
						zi[ q ] = z[ at[ q ] ];
						if( ( flags & 1 ) && i[ q ] >= 0 ) {
							const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ pos[ q ] - pos_begin ] ) );
							zi[ q ] = __dadd_rn( __dmul_rn( 1.0, zi[ q ] ), __dmul_rn( 1.0, f ) );
							z[ i[ q ] ] = zi[ q ];
						}
					}
					const double d = dp.e[ lc.diag_code() ].val;
					const int passes = ( flags & 4 ) ? 2 : 1; // see k_gs_color_packed
					#pragma unroll 1
					for( int pass = 0; pass < passes; ++pass ) {
						if( warp_ragged ) {
							shared_rows_sum< NCODES, CHUNKS, R, true >( lc, z, at, dp, acc );
						} else {
							shared_rows_sum< NCODES, CHUNKS, R, false >( lc, z, at, dp, acc );
						}
						#pragma unroll
						for( int q = 0; q < R; ++q ) {
							zi[ q ] = __ddiv_rn( __dadd_rn( __dadd_rn( ri[ q ], -acc[ q ] ), __dmul_rn( zi[ q ], d ) ), d );
							if( i[ q ] >= 0 ) {
								z[ i[ q ] ] = zi[ q ];
							}
						}
					}
					if( flags & 2 ) {
						if( warp_ragged ) {
							shared_rows_sum< NCODES, CHUNKS, R, true >( lc, z, at, dp, acc );
						} else {
							shared_rows_sum< NCODES, CHUNKS, R, false >( lc, z, at, dp, acc );
						}
						#pragma unroll
						for( int q = 0; q < R; ++q ) {
							if( i[ q ] >= 0 ) {
								const double f = __dadd_rn( __dmul_rn( 1.0, ri[ q ] ), __dmul_rn( -1.0, acc[ q ] ) );
								out[ pos[ q ] - pos_begin ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
								zero[ pos[ q ] - pos_begin ] = 0.0;
							}
						}
					}
					return;
				}
				// rows that differ (grid boundaries, escaped rows, the tail of the range): one at a time
				// (unrolled: indexing the per-row arrays with a run-time q would push them to local memory)
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					if( i[ q ] < 0 ) {
						continue;
					}
					const int64_t coarse = pos[ q ] - pos_begin;
					const double ri = r[ i[ q ] ];
					double zi = z[ i[ q ] ];
					if( flags & 1 ) {
						const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ coarse ] ) );
						zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
						z[ i[ q ] ] = zi;
					}
					const int passes = ( flags & 4 ) ? 2 : 1;
					#pragma unroll 1
					for( int pass = 0; pass < passes; ++pass ) {
						double d = 0.0;
						const double sum = any_row_sum< NCODES, CHUNKS, 1, true >( rc[ q ], true, plain, pos[ q ], i[ q ], z, dp, d );
						zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -sum ), __dmul_rn( zi, d ) ), d );
						z[ i[ q ] ] = zi;
					}
					if( flags & 2 ) {
						double unused = 0.0;
						const double az = any_row_sum< NCODES, CHUNKS, 1, false >( rc[ q ], true, plain, pos[ q ], i[ q ], z, dp, unused );
						const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
						out[ coarse ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
						zero[ coarse ] = 0.0;
					}
				}
			}

			// k_spmv_packed (unmasked) with R rows per thread
			template< int NCODES, int CHUNKS, int R, int DICT >
			__global__ void __launch_bounds__( kBlock ) k_spmv_packed_multi( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, int stride, const double * x, double * y, int64_t count,
				double * dot_partials ) {
				__shared__ double smem[ 32 ];
				const int lane = threadIdx.x & 31;
				const unsigned int gw = ( blockIdx.x * blockDim.x + threadIdx.x ) >> 5;
				const int64_t slice0 = multi_first_slice< R >( 0, gw, static_cast< unsigned int >( stride ) );
				int64_t row[ R ];
				bool live[ R ];
				RowCodes< CHUNKS > rc[ R ];
				#pragma unroll
				for( int q = 0; q < R; ++q ) {
					row[ q ] = ( slice0 + static_cast< int64_t >( q ) * stride ) * kSlice + lane;
					live[ q ] = row[ q ] < count;
					#pragma unroll
					for( int j = 0; j < CHUNKS; ++j ) {
						rc[ q ].q[ j ] = make_uint4( 0u, 0u, 0u, 0u );
					}
					if( live[ q ] ) {
						codes_load( codes, row[ q ], rc[ q ] );
					}
				}
				dep_trigger();
				dep_wait();
				bool same = live[ 0 ] && !rc[ 0 ].escaped();
				#pragma unroll
				for( int q = 1; q < R; ++q ) {
					same = same && live[ q ] && same_codes( rc[ q ], rc[ 0 ] );
				}
				const bool shared = __all_sync( 0xffffffffu, same );
				const bool warp_ragged = __any_sync( 0xffffffffu, rc[ 0 ].template ragged< NCODES >() );
				double prod = 0.0;
				if( shared ) {
					double acc[ R ];
					int32_t row32[ R ];
					#pragma unroll
					for( int q = 0; q < R; ++q ) {
						row32[ q ] = static_cast< int32_t >( row[ q ] );
					}
					if( warp_ragged ) {
						shared_rows_sum< NCODES, CHUNKS, R, true >( rc[ 0 ], x, row32, dp, acc );
					} else {
						shared_rows_sum< NCODES, CHUNKS, R, false >( rc[ 0 ], x, row32, dp, acc );
					}
					#pragma unroll
					for( int q = 0; q < R; ++q ) {
						y[ row[ q ] ] = acc[ q ];
						if( dot_partials != nullptr ) { // the thread's rows in ascending order
							prod = __dadd_rn( prod, __dmul_rn( x[ row[ q ] ], acc[ q ] ) );
						}
					}
				} else {
					#pragma unroll
					for( int q = 0; q < R; ++q ) {
						if( !live[ q ] ) {
							continue;
						}
						double unused = 0.0;
						const double acc = any_row_sum< NCODES, CHUNKS, 1, false >( rc[ q ], true, plain, row[ q ], static_cast< int32_t >( row[ q ] ), x, dp, unused );
						y[ row[ q ] ] = acc;
						if( dot_partials != nullptr ) {
							prod = __dadd_rn( prod, __dmul_rn( x[ row[ q ] ], acc ) );
						}
					}
				}
				if( dot_partials != nullptr ) {
					const double block_sum = block_tree_sum( prod, smem );
					if( threadIdx.x == 0 ) {
						dot_partials[ blockIdx.x ] = block_sum;
					}
				}
			}

			// how often do the rows `s` slices apart carry the same codes? votes[s], s = 1..kMaxStride, over a
			// sample of the slices; votes[0] counts the sampled rows
			constexpr int kMaxStride = 32;
			__global__ void __launch_bounds__( kBlock ) k_stride_votes( const uint4 * __restrict__ codes, int chunks, int64_t nslices,
				int sample_every, unsigned long long * votes ) {
				__shared__ unsigned int local[ kMaxStride + 1 ];
				for( int t = threadIdx.x; t <= kMaxStride; t += blockDim.x ) {
					local[ t ] = 0u;
				}
				__syncthreads();
				const int64_t k = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				const int64_t slice = ( k >> 5 ) * sample_every;
				const int lane = static_cast< int >( k & 31 );
				if( slice < nslices ) {
					uint4 mine[ kMaxChunks ];
					bool empty = true;
					for( int j = 0; j < chunks; ++j ) {
						mine[ j ] = codes[ ( slice * chunks + j ) * kSlice + lane ];
						empty = empty && ( mine[ j ].x | mine[ j ].y | mine[ j ].z | mine[ j ].w ) == 0u;
					}
					if( !empty ) {
						atomicAdd( &local[ 0 ], 1u );
						for( int s = 1; s <= kMaxStride; ++s ) {
							if( slice + s >= nslices ) {
								break;
							}
							bool equal = true;
							for( int j = 0; j < chunks; ++j ) {
								const uint4 other = codes[ ( ( slice + s ) * chunks + j ) * kSlice + lane ];
								equal = equal && other.x == mine[ j ].x && other.y == mine[ j ].y && other.z == mine[ j ].z && other.w == mine[ j ].w;
							}
							if( equal ) {
								atomicAdd( &local[ s ], 1u );
							}
						}
					}
				}
				__syncthreads();
				for( int t = threadIdx.x; t <= kMaxStride; t += blockDim.x ) {
					if( local[ t ] != 0u ) {
						atomicAdd( votes + t, static_cast< unsigned long long >( local[ t ] ) );
					}
				}
			}

			// ------------------------------------------------------------ dispatch on the width class

			// batch: words (of 4 codes) whose gathers are in flight together; dictionary capacity of the
			// parameter block: 32 entries (384 bytes) when that is enough, else all 256 (3 KB)
			template< int N, int D, class F >
			void by_batch( F && f ) {
				constexpr int C = ( N + 16 ) / 16;
				constexpr int W = ( N + 3 ) / 4;
				if( g_packed_batch >= 2 && W > 2 ) {
					f( std::integral_constant< int, N >(), std::integral_constant< int, C >(), std::integral_constant< int, 2 >(),
						std::integral_constant< int, D >() );
				} else {
					f( std::integral_constant< int, N >(), std::integral_constant< int, C >(), std::integral_constant< int, 1 >(),
						std::integral_constant< int, D >() );
				}
			}
			template< int D, class F >
			void by_width( int ncodes, F && f ) {
				switch( ncodes ) {
					case 8: by_batch< 8, D >( f ); break;
					case 16: by_batch< 16, D >( f ); break;
					case 27: by_batch< 27, D >( f ); break;
					case 32: by_batch< 32, D >( f ); break;
					case 64: by_batch< 64, D >( f ); break;
					default: fail( SLAB_ERR_INTERNAL, "packed matrix with an unknown width class" );
				}
			}
			template< class F >
			void by_shape( const Packed & P, F && f ) {
				if( P.dict_size <= 32 ) {
					by_width< 32 >( P.ncodes, f );
				} else {
					by_width< 256 >( P.ncodes, f );
				}
			}
			template< int DICT >
			DictParam< DICT > dict_param( const Packed & P ) {
				DictParam< DICT > dp;
				for( int t = 0; t < DICT; ++t ) {
					dp.e[ t ].val = t < P.dict_size ? P.h_dict[ t ].val : 0.0;
					dp.e[ t ].delta = t < P.dict_size ? P.h_dict[ t ].delta : 0;
				}
				return dp;
			}

			// rows per thread of the multi-row kernels
			template< int D, class F >
			void by_width_rows( int ncodes, int rows_per_thread, F && f ) {
				const auto go = [ & ]( auto N ) {
					constexpr int C = ( N.value + 16 ) / 16;
					if( rows_per_thread >= 4 ) {
						f( N, std::integral_constant< int, C >(), std::integral_constant< int, 4 >(), std::integral_constant< int, D >() );
					} else if( rows_per_thread == 3 ) {
						f( N, std::integral_constant< int, C >(), std::integral_constant< int, 3 >(), std::integral_constant< int, D >() );
					} else {
						f( N, std::integral_constant< int, C >(), std::integral_constant< int, 2 >(), std::integral_constant< int, D >() );
					}
				};
				switch( ncodes ) {
					case 8: go( std::integral_constant< int, 8 >() ); break;
					case 16: go( std::integral_constant< int, 16 >() ); break;
					case 27: go( std::integral_constant< int, 27 >() ); break;
					case 32: go( std::integral_constant< int, 32 >() ); break;
					case 64: go( std::integral_constant< int, 64 >() ); break;
					default: fail( SLAB_ERR_INTERNAL, "packed matrix with an unknown width class" );
				}
			}
			template< class F >
			void by_shape_rows( const Packed & P, int rows_per_thread, F && f ) {
				if( P.dict_size <= 32 ) {
					by_width_rows< 32 >( P.ncodes, rows_per_thread, f );
				} else {
					by_width_rows< 256 >( P.ncodes, rows_per_thread, f );
				}
			}
			bool multi_for( const Packed & P, int rows_per_thread, int64_t rows ) {
				return rows_per_thread >= 2 && P.stride > 0 && rows >= g_packed_multi_min_rows;
			}
			// warps (and from them blocks) a multi-row launch over `nslices` slices needs
			unsigned int multi_grid( int64_t nslices, int rows_per_thread, int stride, int block ) {
				const int64_t tile = static_cast< int64_t >( rows_per_thread ) * stride;
				const int64_t tiles = ( nslices + tile - 1 ) / tile;
				const int64_t warps = tiles * stride;
				return blocks_for( static_cast< uint64_t >( warps ) * 32u, block );
			}

			int block_size() {
				return g_packed_block == 128 ? 128 : 256;
			}

		} // namespace

		void spmv_packed( cudaStream_t st, const Sell & S, const double * x, double * y, const int32_t * members,
			int64_t count, double * dot_partials, double * dot_out ) {
			const Packed & P = S.packed;
			const PlainRef plain{ S.slice_off, S.vals, S.cols };
			const int block = block_size();
			if( members == nullptr && multi_for( P, g_packed_rows_spmv, count ) ) {
				unsigned int grid = 0;
				by_shape_rows( P, g_packed_rows_spmv, [ & ]( auto N, auto C, auto R, auto D ) {
					grid = multi_grid( ( count + kSlice - 1 ) / kSlice, R.value, P.stride, block );
					launch_pdl( k_spmv_packed_multi< N.value, C.value, R.value, D.value >, grid, block, st, P.codes,
						dict_param< D.value >( P ), plain, P.stride, x, y, count, dot_out != nullptr ? dot_partials : nullptr );
				} );
				if( dot_out != nullptr ) {
					sum_partials( st, dot_partials, grid, dot_out );
				}
				return;
			}
			const unsigned int grid = blocks_for( count, block );
			by_shape( P, [ & ]( auto N, auto C, auto B, auto D ) {
				const auto dp = dict_param< D.value >( P );
				if( members != nullptr ) {
					launch_pdl( k_spmv_packed< N.value, C.value, B.value, true, D.value >, grid, block, st, P.codes, dp, plain,
						x, y, members, count, static_cast< double * >( nullptr ) );
				} else {
					launch_pdl( k_spmv_packed< N.value, C.value, B.value, false, D.value >, grid, block, st, P.codes, dp, plain,
						x, y, members, count, dot_out != nullptr ? dot_partials : nullptr );
				}
			} );
			if( members == nullptr && dot_out != nullptr ) {
				sum_partials( st, dot_partials, grid, dot_out );
			}
		}

		void gs_color_step_packed( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t pos_begin, int64_t pos_count,
			double * z, const double * r, int flags, const double * src, double * out, double * zero, const int32_t * pos_list,
			const uint8_t * skip ) {
			const Packed & P = S.packed;
			const PlainRef plain{ S.slice_off, S.vals, S.cols };
			const int block = block_size();
			if( pos_list == nullptr && skip != nullptr && ( pos_begin % kSlice ) == 0 && multi_for( P, g_packed_rows, pos_count ) ) {
				by_shape_rows( P, g_packed_rows, [ & ]( auto N, auto C, auto R, auto D ) {
					launch_pdl( k_gs_color_packed_multi_skip< N.value, C.value, R.value, D.value >,
						multi_grid( ( pos_count + kSlice - 1 ) / kSlice, R.value, P.stride, block ), block, st, P.codes,
						dict_param< D.value >( P ), plain, rows, P.stride, pos_begin, pos_count, z, r, flags, src, out, zero, skip );
				} );
				return;
			}
			if( pos_list == nullptr && skip == nullptr && ( pos_begin % kSlice ) == 0 && multi_for( P, g_packed_rows, pos_count ) ) {
				by_shape_rows( P, g_packed_rows, [ & ]( auto N, auto C, auto R, auto D ) {
					launch_pdl( k_gs_color_packed_multi< N.value, C.value, R.value, D.value >,
						multi_grid( ( pos_count + kSlice - 1 ) / kSlice, R.value, P.stride, block ), block, st, P.codes,
						dict_param< D.value >( P ), plain, rows, P.stride, pos_begin, pos_count, z, r, flags, src, out, zero );
				} );
				return;
			}
			by_shape( P, [ & ]( auto N, auto C, auto B, auto D ) {
				launch_pdl( k_gs_color_packed< N.value, C.value, B.value, D.value >, blocks_for( pos_count, block ), block, st, P.codes,
					dict_param< D.value >( P ), plain, rows, pos_begin, pos_count, z, r, flags, src, out, zero, pos_list, skip );
			} );
		}

		void residual_restrict_packed( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t n_coarse, const double * z,
			const double * r, double * r_c, double * zero ) {
			const Packed & P = S.packed;
			const PlainRef plain{ S.slice_off, S.vals, S.cols };
			const int block = block_size();
			by_shape( P, [ & ]( auto N, auto C, auto B, auto D ) {
				launch_pdl( k_residual_restrict_packed< N.value, C.value, B.value, D.value >, blocks_for( n_coarse, block ), block, st,
					P.codes, dict_param< D.value >( P ), plain, rows, n_coarse, z, r, r_c, zero );
			} );
		}

	} // namespace kern

	// ---------------------------------------------------------------- building the packed copy

	void sell_pack( slab_ctx_s * ctx, Sell & S, const int32_t * d_rows, int64_t owned_cols ) {
		using namespace kern;
		S.packed.release();
		const int ncodes = width_class( S.max_width );
		if( !g_pack_build || S.nrows == 0 || S.entries == 0 || S.max_width < 1 || ncodes == 0 ) {
			return;
		}
		Packed P;
		P.max_width = S.max_width;
		P.ncodes = ncodes;
		P.chunks = ( ncodes + 16 ) / 16;
		const int64_t npadded = S.nslices * kSlice;
		constexpr unsigned int kCandCap = 2048;
		unsigned long long * d_escaped = nullptr;
		unsigned long long * d_cand_key = nullptr;
		double * d_cand_val = nullptr;
		int32_t * d_cand_delta = nullptr;
		unsigned int * d_cand_hits = nullptr;
		cudaStream_t st = ctx->stream;
		try {
			SLAB_CUDA( cudaMalloc( &P.codes, static_cast< size_t >( npadded ) * P.chunks * sizeof( uint4 ) ) );
			SLAB_CUDA( cudaMalloc( &P.dict, kDict * sizeof( DictEntry ) ) );
			SLAB_CUDA( cudaMalloc( &d_escaped, sizeof( unsigned long long ) ) );
			SLAB_CUDA( cudaMalloc( &d_cand_key, kCandCap * sizeof( unsigned long long ) ) );
			SLAB_CUDA( cudaMalloc( &d_cand_val, kCandCap * sizeof( double ) ) );
			SLAB_CUDA( cudaMalloc( &d_cand_delta, kCandCap * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_cand_hits, kCandCap * sizeof( unsigned int ) ) );
			std::vector< DictEntry > dict( kDict, DictEntry{ 0.0, 0, 0 } );
			std::set< std::pair< int32_t, uint64_t > > known;
			int dict_size = 1; // entry 0: padding
			unsigned long long escaped = 0;
			for( int round = 0;; ++round ) {
				upload_sync( st, P.dict, dict.data(), kDict * sizeof( DictEntry ) );
				SLAB_CUDA( cudaMemsetAsync( d_escaped, 0, sizeof( unsigned long long ), st ) );
				SLAB_CUDA( cudaMemsetAsync( d_cand_key, 0, kCandCap * sizeof( unsigned long long ), st ) );
				SLAB_CUDA( cudaMemsetAsync( d_cand_hits, 0, kCandCap * sizeof( unsigned int ), st ) );
				k_pack_rows<<< dev::blocks_for( npadded ), dev::kBlock, 0, st >>>( S.slice_off, S.vals, S.cols, d_rows, S.nrows, npadded,
					P.dict, dict_size, P.chunks, P.codes, d_escaped, d_cand_key, kCandCap, d_cand_val, d_cand_delta, d_cand_hits,
					static_cast< int32_t >( owned_cols < 0 || owned_cols > 0x7fffffff ? 0x7fffffff : owned_cols ) );
				SLAB_CUDA( cudaGetLastError() );
				count_launch();
				SLAB_CUDA( cudaMemcpyAsync( &escaped, d_escaped, sizeof( escaped ), cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaStreamSynchronize( st ) );
				if( escaped == 0 || round == 7 || dict_size == kDict - 1 ) {
					break;
				}
				std::vector< unsigned long long > ck( kCandCap );
				std::vector< double > cv( kCandCap );
				std::vector< int32_t > cd( kCandCap );
				std::vector< unsigned int > ch( kCandCap );
				SLAB_CUDA( cudaMemcpyAsync( ch.data(), d_cand_hits, kCandCap * sizeof( unsigned int ), cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaMemcpyAsync( ck.data(), d_cand_key, kCandCap * sizeof( unsigned long long ), cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaMemcpyAsync( cv.data(), d_cand_val, kCandCap * sizeof( double ), cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaMemcpyAsync( cd.data(), d_cand_delta, kCandCap * sizeof( int32_t ), cudaMemcpyDeviceToHost, st ) );
				SLAB_CUDA( cudaStreamSynchronize( st ) );
				// new pairs, the most frequent first (then narrow bands first, for a reproducible order): when the
				// dictionary cannot hold everything, the pairs that occur once (ghost slots of a decomposed level)
				// are the ones left to the plain path
				struct Fresh {
					unsigned int hits;
					int32_t delta;
					uint64_t bits;
				};
				std::vector< Fresh > fresh;
				std::set< std::pair< int32_t, uint64_t > > seen;
				for( unsigned int t = 0; t < kCandCap; ++t ) {
					if( ck[ t ] == 0ull ) {
						continue;
					}
					uint64_t bits;
					std::memcpy( &bits, &cv[ t ], sizeof( bits ) );
					const std::pair< int32_t, uint64_t > key( cd[ t ], bits );
					if( !known.count( key ) && seen.insert( key ).second ) {
						fresh.push_back( Fresh{ ch[ t ], cd[ t ], bits } );
					}
				}
				std::sort( fresh.begin(), fresh.end(), []( const Fresh & a, const Fresh & b ) {
					if( a.hits != b.hits ) {
						return a.hits > b.hits;
					}
					const int64_t da = a.delta < 0 ? -static_cast< int64_t >( a.delta ) : a.delta;
					const int64_t db = b.delta < 0 ? -static_cast< int64_t >( b.delta ) : b.delta;
					return da != db ? da < db : ( a.delta != b.delta ? a.delta < b.delta : a.bits < b.bits );
				} );
				bool grew = false;
				for( const Fresh & f : fresh ) {
					if( dict_size >= kDict - 1 ) {
						break;
					}
					known.insert( std::make_pair( f.delta, f.bits ) );
					dict[ dict_size ].delta = f.delta;
					std::memcpy( &dict[ dict_size ].val, &f.bits, sizeof( double ) );
					++dict_size;
					grew = true;
				}
				if( !grew ) {
					break;
				}
			}
			P.dict_size = dict_size;
			P.escaped_rows = static_cast< int64_t >( escaped );
			P.h_dict = new DictEntry[ kDict ];
			std::copy( dict.begin(), dict.end(), P.h_dict );
		} catch( ... ) {
			cudaFree( d_escaped );
			cudaFree( d_cand_key );
			cudaFree( d_cand_val );
			cudaFree( d_cand_delta );
			cudaFree( d_cand_hits );
			P.release();
			throw;
		}
		cudaFree( d_escaped );
		cudaFree( d_cand_key );
		cudaFree( d_cand_val );
		cudaFree( d_cand_delta );
		cudaFree( d_cand_hits );
		if( std::getenv( "SLAB_PACK_DEBUG" ) ) {
			std::fprintf( stderr, "sell_pack: nrows %lld max_width %d dict %d escaped %lld\n", static_cast< long long >( S.nrows ),
				S.max_width, P.dict_size, static_cast< long long >( P.escaped_rows ) );
		}
		// not worth it when many rows would take the plain path anyway (each costs both code paths)
		if( P.escaped_rows * 8 > S.nrows ) {
			P.release();
			return;
		}
		// the slice distance at which rows most often repeat their codes (multi-row kernels)
		{
			unsigned long long * d_votes = nullptr;
			unsigned long long votes[ kMaxStride + 1 ] = { 0 };
			const int sample_every = S.nslices > 4096 ? 8 : 1;
			const int64_t sampled = ( S.nslices + sample_every - 1 ) / sample_every;
			SLAB_CUDA( cudaMalloc( &d_votes, sizeof( votes ) ) );
			SLAB_CUDA( cudaMemsetAsync( d_votes, 0, sizeof( votes ), st ) );
			k_stride_votes<<< dev::blocks_for( sampled * kSlice ), dev::kBlock, 0, st >>>( P.codes, P.chunks, S.nslices, sample_every, d_votes );
			count_launch();
			const cudaError_t err = cudaMemcpyAsync( votes, d_votes, sizeof( votes ), cudaMemcpyDeviceToHost, st );
			const cudaError_t err2 = cudaStreamSynchronize( st );
			cudaFree( d_votes );
			if( err != cudaSuccess || err2 != cudaSuccess ) {
				P.release();
				SLAB_CUDA( err != cudaSuccess ? err : err2 );
			}
			int best = 0;
			for( int t = 1; t <= kMaxStride; ++t ) {
				if( votes[ t ] > ( best ? votes[ best ] : 0ull ) ) {
					best = t;
				}
			}
			P.stride = ( best > 0 && votes[ best ] * 4 >= votes[ 0 ] * 3 ) ? best : 0; // at least 3 rows in 4 repeat
		}
		S.packed = P;
		if( !g_keep_plain && P.escaped_rows == 0 ) {
			cudaFree( S.vals );
			cudaFree( S.cols );
			S.vals = nullptr;
			S.cols = nullptr;
		}
	}

} // namespace slabgpu
