// packed_decode.cuh — device-side decoder of the dictionary-coded SELL rows (format: packed.cu's header comment),
// shared by the translation units that read coded matrices (packed.cu, sweep_cluster.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"

namespace slabgpu {
	namespace kern {
		namespace coded {

			using namespace dev;

			constexpr unsigned int kEscape = 255u;

			// ------------------------------------------------------------ decoder

			template< int CHUNKS >
			struct RowCodes {
				uint4 q[ CHUNKS ];
				__device__ __forceinline__ unsigned int word( int wi ) const {
					const uint4 & v = q[ wi >> 2 ];
					switch( wi & 3 ) {
						case 0: return v.x;
						case 1: return v.y;
						case 2: return v.z;
						default: return v.w;
					}
				}
				__device__ __forceinline__ bool escaped() const {
					return ( q[ 0 ].x & 0xffu ) == kEscape;
				}
				__device__ __forceinline__ unsigned int diag_code() const {
					return q[ CHUNKS - 1 ].w >> 24;
				}
				// does any of the first NCODES codes say "padding"? (rows narrower than the width class)
				template< int NCODES >
				__device__ __forceinline__ bool ragged() const {
					constexpr int WORDS = ( NCODES + 3 ) / 4;
					unsigned int hit = 0u;
					#pragma unroll
					for( int wi = 0; wi < WORDS; ++wi ) {
						unsigned int w = word( wi );
						if( wi == WORDS - 1 && ( NCODES & 3 ) != 0 ) {
							w |= 0xffffffffu << ( 8 * ( NCODES & 3 ) );
						}
						hit |= ( w - 0x01010101u ) & ~w & 0x80808080u; // non-zero iff some byte of w is zero
					}
					return hit != 0u;
				}
			};

			template< int CHUNKS >
			__device__ __forceinline__ void codes_load( const uint4 * __restrict__ codes, int64_t pos, RowCodes< CHUNKS > & rc ) {
				const uint4 * p = codes + ( ( pos >> 5 ) * CHUNKS ) * kSlice + ( pos & 31 );
				#pragma unroll
				for( int j = 0; j < CHUNKS; ++j ) {
					rc.q[ j ] = __ldcs( p + j * kSlice );
				}
			}

			// The dictionary travels as a kernel parameter and is read with indexed constant loads: the 32
			// rows of an interior slice carry the same codes, so the index is warp-uniform and the read costs
			// one constant-cache access — unlike a shared-memory table, it takes nothing from the L1 data
			// pipe, which the gathers saturate (measured: shared-memory lookups were 45% of its wavefronts).
			template< int DICT >
			struct DictParam { // value and offset of a code side by side: one index computation serves both reads
				struct Entry {
					double val;
					int32_t delta;
					int32_t unused;
				} e[ DICT ];
			};

			// ordered row sum over the coded entries: acc = acc + val*xrow[delta] (xrow = x + row), ascending
			// column order. RAGGED rows test every code for padding (code 0 is skipped); full rows do not.
			// The gathers of BATCH 4-code words go out before their add chain runs: a large BATCH suits
			// latency-bound small launches (every gather of the row in flight at once), a small one keeps
			// the register count low for many-wave launches.
			template< int NCODES, int CHUNKS, int BATCH, bool RAGGED, int DICT >
			__device__ __forceinline__ double coded_row_sum( const RowCodes< CHUNKS > & rc, const double * xrow,
				const DictParam< DICT > & dp ) {
				constexpr int WORDS = ( NCODES + 3 ) / 4;
				double acc = 0.0;
				#pragma unroll
				for( int w0 = 0; w0 < WORDS; w0 += BATCH ) {
					double xv[ 4 * BATCH ];
					#pragma unroll
					for( int b = 0; b < BATCH; ++b ) {
						#pragma unroll
						for( int j = 0; j < 4; ++j ) {
							if( 4 * ( w0 + b ) + j < NCODES ) {
								const unsigned int code = ( rc.word( w0 + b ) >> ( 8 * j ) ) & 0xffu;
								xv[ 4 * b + j ] = xrow[ dp.e[ code ].delta ];
							}
						}
					}
					// keep the batch's gathers together, ahead of the add chain: the assembler schedules within
					// basic blocks, so a never-taken branch pins them (an empty asm only pins the front end)
					if( BATCH > 1 ) {
						asm volatile( "" ::: "memory" );
						if( dp.e[ 0 ].delta == 0x7fffffff ) { // entry 0 is {0.0, 0}
							__trap();
						}
					}
					#pragma unroll
					for( int b = 0; b < BATCH; ++b ) {
						#pragma unroll
						for( int j = 0; j < 4; ++j ) {
							if( 4 * ( w0 + b ) + j < NCODES ) {
								const unsigned int code = ( rc.word( w0 + b ) >> ( 8 * j ) ) & 0xffu;
								const double prod = __dmul_rn( dp.e[ code ].val, xv[ 4 * b + j ] );
								if( !RAGGED || code != 0u ) { // a predicated add, not a select: padding adds nothing
									acc = __dadd_rn( acc, prod );
								}
							}
						}
					}
				}
				return acc;
			}

			// the same sum for an escaped row, from the plain SELL arrays
			template< bool WANT_DIAG >
			__device__ __noinline__ double plain_row_sum( const int64_t * __restrict__ slice_off, const double * __restrict__ vals,
				const int32_t * __restrict__ cols, int64_t pos, const double * x, int32_t diag_row, double & diag ) {
				const int64_t s = pos >> 5;
				const int64_t begin = slice_off[ s ] + ( pos & 31 );
				const int64_t end = slice_off[ s + 1 ];
				double acc = 0.0;
				for( int64_t e = begin; e < end; e += kSlice ) {
					const int32_t c = cols[ e ];
					const double v = vals[ e ];
					if( c >= 0 ) {
						acc = __dadd_rn( acc, __dmul_rn( v, x[ c ] ) );
						if( WANT_DIAG && c == diag_row ) {
							diag = v;
						}
					}
				}
				return acc;
			}

			struct PlainRef { // the plain arrays, for escaped rows
				const int64_t * slice_off;
				const double * vals;
				const int32_t * cols;
			};

			// row sum of any packed row: escaped -> plain arrays (rare, divergent); otherwise the warp takes
			// ONE path — the padding-testing one if any of its rows is narrower than the width class, the
			// test-free one if none is (`warp_ragged` is a warp vote taken by the caller)
			template< int NCODES, int CHUNKS, int BATCH, bool WANT_DIAG, int DICT >
			__device__ __forceinline__ double any_row_sum( const RowCodes< CHUNKS > & rc, bool warp_ragged, const PlainRef & plain,
				int64_t pos, int32_t row, const double * x, const DictParam< DICT > & dp, double & diag ) {
				if( rc.escaped() ) {
					return plain_row_sum< WANT_DIAG >( plain.slice_off, plain.vals, plain.cols, pos, x, row, diag );
				}
				if( WANT_DIAG ) {
					diag = dp.e[ rc.diag_code() ].val;
				}
				if( warp_ragged ) {
					return coded_row_sum< NCODES, CHUNKS, BATCH, true >( rc, x + row, dp );
				}
				return coded_row_sum< NCODES, CHUNKS, BATCH, false >( rc, x + row, dp );
			}

		} // namespace coded
	} // namespace kern
} // namespace slabgpu
