// sweep_cluster.cu — a whole symmetric Gauss-Seidel sweep of a SMALL level in one launch (experiment, off by default).
//
// Why. A colour step of a coarse level is a few hundred to a few thousand rows: its kernel runs at the floor
// of a dependent launch (2.2 us on B200 inside a CUDA graph with programmatic launches), and a symmetric sweep
// is fifteen of them (smoother.hpp:108-111). Here one thread-block cluster (up to 16 CTAs, one row per thread)
// walks the colours of the sweep itself and separates them with the cluster's hardware barrier
// (barrier.cluster, release/acquire at cluster scope) instead of a kernel boundary. Everything a row needs that
// the sweep does not change — its codes, its row index, r[i] — sits in shared memory from the prologue on, so a
// phase is barrier -> one round of gathers from the L2 -> the row's add chain -> store -> barrier.
//
// Same arithmetic per row, same colour order as the per-colour launches (k_gs_color_packed in packed.cu):
// rows of one colour do not read each other (coloring.hpp:114-158), so the order of rows inside a colour is
// free and the iterates are bit-identical (tests/test_gpu_cluster_sweep.py). The grid transfers ride on the
// first and last step exactly as they do there (flags bit 0 / bit 1).
//
// Measured (tools/cluster_sweep_probe.py, tools/solve_sweep.py --sets cluster_rows=...): a phase costs 2.1-2.6 us,
// i.e. what a launch costs — 64^3 solve 14.08 -> 13.84 ms with levels 2-3 on this path, 192^3 57.0 -> 58.8 ms.
// The ncu source page puts the stall on ERRBAR/UCGABAR_WAIT: publishing z through GLOBAL memory makes every
// `arrive.release` a device-wide memory barrier, which costs as much as the kernel boundary it replaces. The
// version worth building keeps z in (distributed) shared memory, where the cluster barrier alone orders the
// accesses. Until then the per-colour launches stay the default: tuning key "cluster_rows" = 0.
#include "kernels.cuh"

#include <algorithm>
#include <type_traits>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"
#include "packed_decode.cuh"

namespace slabgpu {

	// largest colour (rows) of a level that takes the cluster sweep (at most 16 CTAs x 256 threads, one row per
	// thread); 0 = off, the default (see above)
	int64_t g_cluster_rows = 0;

	namespace kern {

		namespace {

			using namespace dev;
			using namespace coded;

			constexpr int kMaxSweepColors = 8;
			constexpr int kMaxClusterCtas = 16;
			constexpr int kMaxSweepSmem = 200 * 1024;

			size_t sweep_smem_bytes( int ncolors, int chunks, unsigned int block ) {
				return static_cast< size_t >( ncolors ) * block * ( 16u * chunks + 8u + 4u );
			}

			struct SweepColors {
				int32_t pos[ kMaxSweepColors ];   // first position of the colour in the colour-sorted matrix
				int32_t count[ kMaxSweepColors ]; // members
				int32_t ncolors;
			};

			__device__ __forceinline__ void cluster_arrive() {
				asm volatile( "barrier.cluster.arrive.release;" ::: "memory" );
			}
			__device__ __forceinline__ void cluster_wait() {
				asm volatile( "barrier.cluster.wait.acquire;" ::: "memory" );
			}

			// Shared memory of a CTA: what its rows need and the sweep does not change — codes, row index, r[i] — for
			// every colour, one slot per thread: [colour][chunk][thread] uint4 | [colour][thread] double | [colour][thread] int32.
			// Filled once in the prologue (the matrix part before the wait on the previous kernel), so that a phase is
			// barrier -> one round of gathers from the L2 -> the row's add chain -> store -> barrier and nothing else.
			extern __shared__ uint4 sweep_smem[];

			// steps of the sweep: colours 0..nc-1, then nc-2..0; the step of colour nc-1 applies its update twice
			// (the last colour of the forward sweep is the first of the backward sweep, smoother.hpp:108-111)
			template< int NCODES, int CHUNKS, int BATCH, int DICT >
			__global__ void __launch_bounds__( kBlock ) k_gs_sweep_cluster( const uint4 * __restrict__ codes,
				const __grid_constant__ DictParam< DICT > dp, PlainRef plain, const int32_t * __restrict__ rows,
				const __grid_constant__ SweepColors sc, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				const int tx = static_cast< int >( threadIdx.x );
				const int B = static_cast< int >( blockDim.x );
				const int t = static_cast< int >( blockIdx.x ) * B + tx;
				const int nc = sc.ncolors;
				const int nsteps = 2 * nc - 1;
				uint4 * s_codes = sweep_smem;
				double * s_r = reinterpret_cast< double * >( s_codes + nc * CHUNKS * B );
				int32_t * s_i = reinterpret_cast< int32_t * >( s_r + nc * B );
				{
					// all loads of all colours go out together (unrolled: a rolled loop would wait for each colour's data
					// before asking for the next)
					int32_t row_of[ kMaxSweepColors ];
					RowCodes< CHUNKS > rc_of[ kMaxSweepColors ];
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						row_of[ c ] = -1;
						if( c < nc && t < sc.count[ c ] ) {
							const int32_t pos = sc.pos[ c ] + t;
							row_of[ c ] = rows != nullptr ? rows[ pos ] : pos;
							codes_load( codes, static_cast< int64_t >( pos ), rc_of[ c ] );
						}
					}
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						if( c < nc ) {
							s_i[ c * B + tx ] = row_of[ c ];
							if( row_of[ c ] >= 0 ) {
								#pragma unroll
								for( int j = 0; j < CHUNKS; ++j ) {
									s_codes[ ( c * CHUNKS + j ) * B + tx ] = rc_of[ c ].q[ j ];
								}
							}
						}
					}
					dep_trigger();
					dep_wait();
					double r_of[ kMaxSweepColors ];
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						r_of[ c ] = c < nc && row_of[ c ] >= 0 ? r[ row_of[ c ] ] : 0.0;
					}
					#pragma unroll
					for( int c = 0; c < kMaxSweepColors; ++c ) {
						if( c < nc ) {
							s_r[ c * B + tx ] = r_of[ c ];
						}
					}
				}
				#pragma unroll 1
				for( int s = 0; s < nsteps; ++s ) {
					const int c = s < nc ? s : nsteps - 1 - s;
					const int32_t i = s_i[ c * B + tx ];
					if( i >= 0 ) {
						RowCodes< CHUNKS > rc;
						#pragma unroll
						for( int j = 0; j < CHUNKS; ++j ) {
							rc.q[ j ] = s_codes[ ( c * CHUNKS + j ) * B + tx ];
						}
						const double ri = s_r[ c * B + tx ];
						const int32_t pos = sc.pos[ c ] + t;
						const int flags = ( s == 0 ? first_flags : 0 ) | ( s == nsteps - 1 ? last_flags : 0 );
						const int passes = s == nc - 1 ? 2 : 1;
						const bool warp_ragged = __any_sync( __activemask(), rc.template ragged< NCODES >() );
						double zi = z[ i ];
						if( flags & 1 ) { // multigrid.hpp:76-77 on the injected rows
							const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ t ] ) );
							zi = __dadd_rn( __dmul_rn( 1.0, zi ), __dmul_rn( 1.0, f ) );
							z[ i ] = zi;
						}
						#pragma unroll 1
						for( int pass = 0; pass < passes; ++pass ) { // smoother.hpp:60-72
							double d = 0.0;
							const double sum = any_row_sum< NCODES, CHUNKS, BATCH, true >( rc, warp_ragged, plain, pos, i, z, dp, d );
							zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -sum ), __dmul_rn( zi, d ) ), d );
							z[ i ] = zi;
						}
						if( flags & 2 ) { // multigrid.hpp:100-104 on the injected rows
							double unused = 0.0;
							const double az = any_row_sum< NCODES, CHUNKS, BATCH, false >( rc, warp_ragged, plain, pos, i, z, dp, unused );
							const double f = __dadd_rn( __dmul_rn( 1.0, ri ), __dmul_rn( -1.0, az ) );
							out[ t ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
							zero[ t ] = 0.0;
						}
					}
					if( s + 1 < nsteps ) {
						cluster_arrive();
						cluster_wait();
					}
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

			template< class... KArgs, class... Args >
			void launch_cluster( void ( *kernel )( KArgs... ), unsigned int ctas, unsigned int block, size_t smem_bytes, cudaStream_t st,
				Args... args ) {
				cudaLaunchConfig_t cfg{};
				cfg.gridDim = dim3( ctas, 1, 1 );
				cfg.blockDim = dim3( block, 1, 1 );
				cfg.dynamicSmemBytes = smem_bytes;
				cfg.stream = st;
				cudaLaunchAttribute attr[ 2 ];
				unsigned int count = 0;
				attr[ count ].id = cudaLaunchAttributeClusterDimension;
				attr[ count ].val.clusterDim.x = ctas;
				attr[ count ].val.clusterDim.y = 1;
				attr[ count ].val.clusterDim.z = 1;
				++count;
				if( g_use_pdl ) {
					attr[ count ].id = cudaLaunchAttributeProgrammaticStreamSerialization;
					attr[ count ].val.programmaticStreamSerializationAllowed = 1;
					++count;
				}
				cfg.attrs = attr;
				cfg.numAttrs = count;
				SLAB_CUDA( cudaLaunchKernelEx( &cfg, kernel, static_cast< KArgs >( args )... ) );
				count_launch();
			}

			template< int N, int D >
			void sweep_launch( cudaStream_t st, const Packed & P, const PlainRef & plain, const int32_t * rows, const SweepColors & sc,
				unsigned int ctas, unsigned int block, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				constexpr int C = ( N + 16 ) / 16;
				constexpr int W = ( N + 3 ) / 4; // every gather of the row in flight at once: the phase is latency-bound
				auto kernel = k_gs_sweep_cluster< N, C, W, D >;
				static bool large_clusters_allowed = false; // clusters of more than 8 CTAs are opt-in per kernel
				if( !large_clusters_allowed ) {
					SLAB_CUDA( cudaFuncSetAttribute( kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1 ) );
					SLAB_CUDA( cudaFuncSetAttribute( kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSweepSmem ) );
					large_clusters_allowed = true;
				}
				launch_cluster( kernel, ctas, block, sweep_smem_bytes( sc.ncolors, C, block ), st, P.codes, dict_param< D >( P ), plain, rows, sc, z, r, first_flags, last_flags,
					src, out, zero );
			}

			template< int D >
			void sweep_by_width( cudaStream_t st, const Packed & P, const PlainRef & plain, const int32_t * rows, const SweepColors & sc,
				unsigned int ctas, unsigned int block, double * z, const double * r, int first_flags, int last_flags,
				const double * src, double * out, double * zero ) {
				switch( P.ncodes ) {
					case 8: sweep_launch< 8, D >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero ); break;
					case 16: sweep_launch< 16, D >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero ); break;
					case 27: sweep_launch< 27, D >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero ); break;
					case 32: sweep_launch< 32, D >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero ); break;
					case 64: sweep_launch< 64, D >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero ); break;
					default: fail( SLAB_ERR_INTERNAL, "packed matrix with an unknown width class" );
				}
			}

		} // namespace

		bool gs_sweep_cluster_usable( const Sell & S, const std::vector< int64_t > & color_pos, const std::vector< uint64_t > & color_size ) {
			if( g_cluster_rows <= 0 || !g_use_packed || !S.packed.usable() ) {
				return false;
			}
			const size_t nc = color_size.size();
			if( nc < 1 || nc > static_cast< size_t >( kMaxSweepColors ) || color_pos.size() < nc ) {
				return false;
			}
			const uint64_t largest = *std::max_element( color_size.begin(), color_size.end() );
			const int64_t limit = std::min< int64_t >( g_cluster_rows, static_cast< int64_t >( kMaxClusterCtas ) * kBlock );
			return largest >= 1 && static_cast< int64_t >( largest ) <= limit && color_pos[ nc - 1 ] < ( int64_t( 1 ) << 30 )
				&& sweep_smem_bytes( static_cast< int >( nc ), S.packed.chunks, kBlock ) <= static_cast< size_t >( kMaxSweepSmem );
		}

		void gs_sweep_cluster( cudaStream_t st, const Sell & S, const int32_t * rows, const std::vector< int64_t > & color_pos,
			const std::vector< uint64_t > & color_size, double * z, const double * r, int first_flags, int last_flags,
			const double * src, double * out, double * zero ) {
			const Packed & P = S.packed;
			const PlainRef plain{ S.slice_off, S.vals, S.cols };
			SweepColors sc{};
			sc.ncolors = static_cast< int32_t >( color_size.size() );
			uint64_t largest = 1;
			for( int k = 0; k < sc.ncolors; ++k ) {
				sc.pos[ k ] = static_cast< int32_t >( color_pos[ k ] );
				sc.count[ k ] = static_cast< int32_t >( color_size[ k ] );
				largest = std::max( largest, color_size[ k ] );
			}
			// spread thin (about 64 rows per CTA: the phase is a latency chain, not a throughput problem), power-of-two clusters
			unsigned int ctas = 1;
			while( ctas < static_cast< unsigned int >( kMaxClusterCtas ) && static_cast< uint64_t >( ctas ) * 64u < largest ) {
				ctas *= 2;
			}
			const unsigned int per_cta = static_cast< unsigned int >( ( largest + ctas - 1 ) / ctas );
			const unsigned int block = std::max( 32u, ( per_cta + 31u ) / 32u * 32u );
			if( P.dict_size <= 32 ) {
				sweep_by_width< 32 >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero );
			} else {
				sweep_by_width< 256 >( st, P, plain, rows, sc, ctas, block, z, r, first_flags, last_flags, src, out, zero );
			}
		}

	} // namespace kern
} // namespace slabgpu
